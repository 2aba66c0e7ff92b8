"""Host-side model graph: the typed DAG the B200 path lowers and runs.

This mirrors the public surface of ``levnet.graph`` (reference
``pkg/src/levnet/graph.py``) so that code written against the reference keeps
working: the same node classes and field names (``graph.py:31-143``), the same
``ModelGraph`` methods (``graph.py:158-249``), the same neutral JSON model
format (``graph.py:433-539``) and the same error types (``graph.py:19-24``).

It adds three node kinds the reference IR cannot express but the benchmark
configurations need:

* ``LocalPoolNode``  -- k x k sum pool with stride/padding times a scalar
  divisor (LeNet 2x2 average pools, the ResNet-18 3x3/s2 stem pool);
  PAPER.md:7-16 treats any average pool as ``divisor * sum``.
* ``FlattenNode``    -- (C, H, W) -> (C*H*W,) in C-major order (LeNet FC1).
* ``BiPoolNode``     -- pairwise bivariate polynomial pool along one spatial
  axis, ``out[c, i] = S(x[c, 2i], x[c, 2i+1])`` with
  ``S(x, y) = sum_{i+j<=d} c_ij x^i y^j``; two of them in
  sequence replace a 2x2 max pool (VGG-11 config).

Nothing in this module computes a forward pass: inference runs on the GPU
(``paper_2509_22857_b200.runtime``).
"""

from __future__ import annotations

import base64
import json
from collections import deque
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np


class GraphError(Exception):
    """A graph invariant does not hold; the message names the node."""


class ModelFormatError(Exception):
    """A model file is not in the neutral format."""


# ---------------------------------------------------------------------------
# node kinds (field names follow reference graph.py:31-143)
# ---------------------------------------------------------------------------

@dataclass
class Node:
    id: str

    @property
    def kind(self) -> str:
        return _KIND_OF[type(self)]


@dataclass
class InputNode(Node):
    channels: int = 1
    height: int = 1
    width: int = 1

    @property
    def shape(self) -> Tuple[int, int, int]:
        return (self.channels, self.height, self.width)


@dataclass
class ConvNode(Node):
    weight: np.ndarray = None  # (O, I, kh, kw)
    bias: np.ndarray = None    # (O,)
    stride: int = 1
    padding: int = 0


@dataclass
class BatchNormNode(Node):
    gamma: np.ndarray = None
    beta: np.ndarray = None
    mean: np.ndarray = None
    std: np.ndarray = None

    @property
    def b1(self) -> np.ndarray:
        """Slope of the affine form B(x) = b1 x + b0 (PAPER.md node fusing)."""
        return self.gamma / self.std

    @property
    def b0(self) -> np.ndarray:
        return self.beta - self.b1 * self.mean


@dataclass
class PolyActNode(Node):
    # coeffs[k] multiplies x^k; each entry has shape () or (C,)
    coeffs: List[np.ndarray] = field(default_factory=list)

    @property
    def degree(self) -> int:
        return len(self.coeffs) - 1

    def is_monic(self) -> bool:
        return bool(np.all(np.asarray(self.coeffs[-1]) == 1.0))


# monomial keys of the quadratic join S(x, y) (reference graph.py:89)
PS_KEYS = ("x2", "y2", "xy", "x", "y", "c")


@dataclass
class PolySkipNode(Node):
    coeffs: Dict[str, np.ndarray] = field(default_factory=dict)

    def is_monic(self) -> bool:
        c = self.coeffs
        return bool(np.all(np.asarray(c["x2"]) == 1.0)
                    and np.all(np.asarray(c["y2"]) == 1.0)
                    and np.all(np.asarray(c["xy"]) == 2.0))


@dataclass
class AvgPoolNode(Node):
    """Global pool: divisor * sum over all H*W positions (k must be H*W)."""
    k: int = 1
    divisor: np.ndarray = None


@dataclass
class LinearNode(Node):
    weight: np.ndarray = None  # (K, n)
    bias: np.ndarray = None    # (K,)


@dataclass
class AddNode(Node):
    pass


@dataclass
class OutputNode(Node):
    pass


# ---- extensions (not in the reference IR) ---------------------------------

@dataclass
class LocalPoolNode(Node):
    """divisor * (k x k window sum), zero padding counted, given stride."""
    k: int = 2
    stride: int = 2
    padding: int = 0
    divisor: np.ndarray = None


@dataclass
class FlattenNode(Node):
    pass


@dataclass
class BiPoolNode(Node):
    """Pairwise bivariate pool along ``axis`` ('w' or 'h').

    ``coeffs[i, j]`` multiplies x^i y^j, where x is the even and y the odd
    element of each pair; shape (d+1, d+1) or (d+1, d+1, C); entries with
    i + j > d must be zero.
    """
    axis: str = "w"
    coeffs: np.ndarray = None

    @property
    def degree(self) -> int:
        return int(np.asarray(self.coeffs).shape[0]) - 1

    def is_monic(self) -> bool:
        d = self.degree
        return bool(np.all(np.asarray(self.coeffs)[d, 0] == 1.0))


_KIND_OF = {
    InputNode: "input", ConvNode: "conv", BatchNormNode: "batchnorm",
    PolyActNode: "polyact", PolySkipNode: "polyskip", AvgPoolNode: "avgpool",
    LinearNode: "linear", AddNode: "add", OutputNode: "output",
    LocalPoolNode: "localpool", FlattenNode: "flatten", BiPoolNode: "bipool",
}
KIND_BY_TYPE = dict(_KIND_OF)
TYPE_BY_KIND = {v: k for k, v in _KIND_OF.items()}

ARITY = {
    "input": 0, "conv": 1, "batchnorm": 1, "polyact": 1, "avgpool": 1,
    "linear": 1, "output": 1, "add": 2, "polyskip": 2,
    "localpool": 1, "flatten": 1, "bipool": 1,
}


def channel_view(coef, ndim: int) -> np.ndarray:
    """Reshape a () or (C,) coefficient to broadcast over a (C, ...) value."""
    a = np.asarray(coef, dtype=np.float64)
    return a if a.ndim == 0 else a.reshape(a.shape + (1,) * (ndim - 1))


def _arr(a) -> np.ndarray:
    return np.array(a, dtype=np.float64)


def copy_node(node: Node) -> Node:
    """Deep copy; every tensor field gets its own float64 storage."""
    if isinstance(node, InputNode):
        return InputNode(node.id, node.channels, node.height, node.width)
    if isinstance(node, ConvNode):
        return ConvNode(node.id, _arr(node.weight), _arr(node.bias), node.stride, node.padding)
    if isinstance(node, BatchNormNode):
        return BatchNormNode(node.id, _arr(node.gamma), _arr(node.beta), _arr(node.mean), _arr(node.std))
    if isinstance(node, PolyActNode):
        return PolyActNode(node.id, [_arr(c) for c in node.coeffs])
    if isinstance(node, PolySkipNode):
        return PolySkipNode(node.id, {k: _arr(v) for k, v in node.coeffs.items()})
    if isinstance(node, AvgPoolNode):
        return AvgPoolNode(node.id, node.k, _arr(node.divisor))
    if isinstance(node, LinearNode):
        return LinearNode(node.id, _arr(node.weight), _arr(node.bias))
    if isinstance(node, LocalPoolNode):
        return LocalPoolNode(node.id, node.k, node.stride, node.padding, _arr(node.divisor))
    if isinstance(node, BiPoolNode):
        return BiPoolNode(node.id, node.axis, _arr(node.coeffs))
    if isinstance(node, (AddNode, OutputNode, FlattenNode)):
        return type(node)(node.id)
    raise GraphError(f"unknown node type {type(node).__name__}")


# ---------------------------------------------------------------------------
# the graph
# ---------------------------------------------------------------------------

class ModelGraph:
    """DAG of typed nodes with ordered edges. A node's fan-in order is the
    order its incoming edges were added (polyskip: x branch first), as in
    reference graph.py:158-160."""

    def __init__(self) -> None:
        self.nodes: Dict[str, Node] = {}
        self.edges: List[Tuple[str, str]] = []

    def add(self, node: Node) -> Node:
        if node.id in self.nodes:
            raise GraphError(f"duplicate node id {node.id!r}")
        self.nodes[node.id] = node
        return node

    def connect(self, src: str, dst: str) -> None:
        self.edges.append((src, dst))

    def inputs_of(self, nid: str) -> List[str]:
        return [s for s, d in self.edges if d == nid]

    def consumers_of(self, nid: str) -> List[str]:
        return [d for s, d in self.edges if s == nid]

    def consumer_edges(self, nid: str) -> List[Tuple[str, int]]:
        """(consumer id, fan-in position) for every out-edge of nid."""
        pos: Dict[str, int] = {}
        out = []
        for s, d in self.edges:
            p = pos.get(d, 0)
            pos[d] = p + 1
            if s == nid:
                out.append((d, p))
        return out

    def copy(self) -> "ModelGraph":
        g = ModelGraph()
        for node in self.nodes.values():
            g.add(copy_node(node))
        g.edges = list(self.edges)
        return g

    def topo_order(self) -> List[str]:
        """Kahn's algorithm seeded in insertion order (same order as the
        reference's list-based walk, graph.py:190-211)."""
        indeg = {nid: 0 for nid in self.nodes}
        succ: Dict[str, List[str]] = {nid: [] for nid in self.nodes}
        for s, d in self.edges:
            if d not in indeg:
                raise GraphError(f"edge references unknown node {d!r}")
            if s not in indeg:
                raise GraphError(f"edge references unknown node {s!r}")
            indeg[d] += 1
            succ[s].append(d)
        ready = deque(nid for nid in self.nodes if indeg[nid] == 0)
        order: List[str] = []
        while ready:
            nid = ready.popleft()
            order.append(nid)
            for d in succ[nid]:
                indeg[d] -= 1
                if indeg[d] == 0:
                    ready.append(d)
        if len(order) != len(self.nodes):
            stuck = sorted(set(self.nodes) - set(order))
            raise GraphError(f"graph has a cycle through {stuck[:3]}")
        return order

    def input_id(self) -> str:
        ids = [n.id for n in self.nodes.values() if isinstance(n, InputNode)]
        if len(ids) != 1:
            raise GraphError(f"expected exactly one input node, found {len(ids)}")
        return ids[0]

    def output_id(self) -> str:
        ids = [n.id for n in self.nodes.values() if isinstance(n, OutputNode)]
        if len(ids) != 1:
            raise GraphError(f"expected exactly one output node, found {len(ids)}")
        return ids[0]

    def validate(self) -> Dict[str, Tuple[int, ...]]:
        """Check every invariant; return the per-node output shape map."""
        order = self.topo_order()
        self.input_id()
        self.output_id()
        fanin: Dict[str, int] = {nid: 0 for nid in self.nodes}
        for _, d in self.edges:
            fanin[d] += 1
        for nid, node in self.nodes.items():
            want = ARITY[node.kind]
            if fanin[nid] != want:
                raise GraphError(
                    f"node {nid!r} ({node.kind}) has fan-in {fanin[nid]}, wants {want}")
        for node in self.nodes.values():
            _check_params(node)
        return self._infer_shapes(order)

    def _infer_shapes(self, order: Optional[List[str]] = None) -> Dict[str, Tuple[int, ...]]:
        preds: Dict[str, List[str]] = {nid: [] for nid in self.nodes}
        for s, d in self.edges:
            preds[d].append(s)
        shapes: Dict[str, Tuple[int, ...]] = {}
        for nid in order or self.topo_order():
            shapes[nid] = _out_shape(self.nodes[nid], [shapes[p] for p in preds[nid]])
        return shapes

    def shapes(self) -> Dict[str, Tuple[int, ...]]:
        return self._infer_shapes()


def _check_params(node: Node) -> None:
    nid = node.id
    if isinstance(node, InputNode):
        if min(node.shape) < 1:
            raise GraphError(f"node {nid!r}: all dimensions must be >= 1")
    elif isinstance(node, ConvNode):
        if node.weight.ndim != 4:
            raise GraphError(f"node {nid!r}: conv weight must be 4-D")
        if node.weight.shape[2] < 1 or node.weight.shape[3] < 1:
            raise GraphError(f"node {nid!r}: kernel dims must be >= 1")
        if node.bias.shape != (node.weight.shape[0],):
            raise GraphError(f"node {nid!r}: bias length != out-channels")
        if node.stride < 1 or node.padding < 0:
            raise GraphError(f"node {nid!r}: stride must be >= 1 and padding >= 0")
    elif isinstance(node, BatchNormNode):
        if not np.all(node.std > 0):
            raise GraphError(f"node {nid!r}: std must be > 0 elementwise")
        n = node.gamma.shape
        if not (node.beta.shape == n and node.mean.shape == n and node.std.shape == n):
            raise GraphError(f"node {nid!r}: batchnorm channel vectors disagree")
    elif isinstance(node, PolyActNode):
        if node.degree < 1:
            raise GraphError(f"node {nid!r}: polynomial degree must be >= 1")
    elif isinstance(node, PolySkipNode):
        if set(node.coeffs) != set(PS_KEYS):
            raise GraphError(f"node {nid!r}: polyskip needs exactly monomials {PS_KEYS}")
    elif isinstance(node, AvgPoolNode):
        if node.k < 1:
            raise GraphError(f"node {nid!r}: pool size must be >= 1")
        if not np.all(np.asarray(node.divisor) > 0):
            raise GraphError(f"node {nid!r}: pool divisor must be > 0")
    elif isinstance(node, LinearNode):
        if node.weight.ndim != 2:
            raise GraphError(f"node {nid!r}: linear weight must be 2-D")
        if node.bias.shape != (node.weight.shape[0],):
            raise GraphError(f"node {nid!r}: bias length != class count")
    elif isinstance(node, LocalPoolNode):
        if node.k < 1 or node.stride < 1 or node.padding < 0 or node.padding >= node.k:
            raise GraphError(f"node {nid!r}: bad local pool window")
        if np.asarray(node.divisor).ndim != 0 or not float(node.divisor) > 0:
            raise GraphError(f"node {nid!r}: pool divisor must be a scalar > 0")
    elif isinstance(node, BiPoolNode):
        c = np.asarray(node.coeffs)
        if c.ndim not in (2, 3) or c.shape[0] != c.shape[1] or c.shape[0] < 2:
            raise GraphError(f"node {nid!r}: bivariate coefficients must be (d+1, d+1[, C])")
        if node.axis not in ("w", "h"):
            raise GraphError(f"node {nid!r}: bivariate pool axis must be 'w' or 'h'")
        d = c.shape[0] - 1
        i, j = np.indices((d + 1, d + 1))
        if np.any(c[(i + j) > d] != 0):
            raise GraphError(f"node {nid!r}: coefficients above total degree {d} must be 0")


def _param_width(node: Node) -> int:
    if isinstance(node, BatchNormNode):
        return node.gamma.shape[0]
    if isinstance(node, BiPoolNode):
        c = np.asarray(node.coeffs)
        return c.shape[2] if c.ndim == 3 else 1
    arrays = node.coeffs if isinstance(node, PolyActNode) else list(node.coeffs.values())
    widths = {np.asarray(a).shape[0] for a in arrays if np.asarray(a).ndim > 0}
    if len(widths) > 1:
        raise GraphError(f"node {node.id!r}: mixed per-channel widths {sorted(widths)}")
    return widths.pop() if widths else 1


def _out_shape(node: Node, ins: List[Tuple[int, ...]]) -> Tuple[int, ...]:
    nid = node.id
    if isinstance(node, InputNode):
        return node.shape
    if isinstance(node, ConvNode):
        if len(ins[0]) != 3:
            raise GraphError(f"node {nid!r}: conv needs a (C, H, W) input")
        c, h, w = ins[0]
        o, i, kh, kw = node.weight.shape
        if i != c:
            raise GraphError(f"node {nid!r}: conv expects {i} channels, got {c}")
        ho = (h + 2 * node.padding - kh) // node.stride + 1
        wo = (w + 2 * node.padding - kw) // node.stride + 1
        if ho < 1 or wo < 1:
            raise GraphError(f"node {nid!r}: kernel larger than padded input")
        return (o, ho, wo)
    if isinstance(node, (BatchNormNode, PolyActNode)):
        width = _param_width(node)
        if width not in (1, ins[0][0]):
            raise GraphError(
                f"node {nid!r}: per-channel params sized {width}, input has {ins[0][0]}")
        return ins[0]
    if isinstance(node, (AddNode, PolySkipNode)):
        if ins[0] != ins[1]:
            raise GraphError(f"node {nid!r}: branch shapes differ {ins[0]} vs {ins[1]}")
        if isinstance(node, PolySkipNode):
            width = _param_width(node)
            if width not in (1, ins[0][0]):
                raise GraphError(
                    f"node {nid!r}: per-channel params sized {width}, input has {ins[0][0]}")
        return ins[0]
    if isinstance(node, AvgPoolNode):
        if len(ins[0]) != 3:
            raise GraphError(f"node {nid!r}: global pool needs a (C, H, W) input")
        c, h, w = ins[0]
        if node.k != h * w:
            raise GraphError(f"node {nid!r}: pool size {node.k} != spatial {h}x{w}")
        return (c,)
    if isinstance(node, LinearNode):
        if len(ins[0]) != 1 or node.weight.shape[1] != ins[0][0]:
            raise GraphError(f"node {nid!r}: linear expects vector of {node.weight.shape[1]}")
        return (node.weight.shape[0],)
    if isinstance(node, LocalPoolNode):
        if len(ins[0]) != 3:
            raise GraphError(f"node {nid!r}: local pool needs a (C, H, W) input")
        c, h, w = ins[0]
        ho = (h + 2 * node.padding - node.k) // node.stride + 1
        wo = (w + 2 * node.padding - node.k) // node.stride + 1
        if ho < 1 or wo < 1:
            raise GraphError(f"node {nid!r}: pool window larger than padded input")
        return (c, ho, wo)
    if isinstance(node, FlattenNode):
        if len(ins[0]) != 3:
            raise GraphError(f"node {nid!r}: flatten needs a (C, H, W) input")
        c, h, w = ins[0]
        return (c * h * w,)
    if isinstance(node, BiPoolNode):
        if len(ins[0]) != 3:
            raise GraphError(f"node {nid!r}: bivariate pool needs a (C, H, W) input")
        c, h, w = ins[0]
        width = _param_width(node)
        if width not in (1, c):
            raise GraphError(f"node {nid!r}: per-channel params sized {width}, input has {c}")
        if node.axis == "w":
            if w % 2:
                raise GraphError(f"node {nid!r}: width {w} is odd")
            return (c, h, w // 2)
        if h % 2:
            raise GraphError(f"node {nid!r}: height {h} is odd")
        return (c, h // 2, w)
    if isinstance(node, OutputNode):
        return ins[0]
    raise GraphError(f"unknown node type {type(node).__name__}")


# ---------------------------------------------------------------------------
# neutral model format (reference graph.py:433-539; extension kinds added)
# ---------------------------------------------------------------------------

FORMAT_VERSION = 1

_TENSORS = {
    "conv": ("weight", "bias"),
    "batchnorm": ("gamma", "beta", "mean", "std"),
    "linear": ("weight", "bias"),
    "avgpool": ("divisor",),
    "localpool": ("divisor",),
    "bipool": ("coeffs",),
}
_PARAMS = {
    "input": ("channels", "height", "width"),
    "conv": ("stride", "padding"),
    "avgpool": ("k",),
    "localpool": ("k", "stride", "padding"),
    "bipool": ("axis",),
}


def save_model(g: ModelGraph, path: str) -> None:
    """Write the neutral JSON format: nodes in topological order, ordered
    edges, every float64 tensor in one little-endian base64 blob referenced
    by {offset (in doubles), shape}."""
    chunks: List[bytes] = []
    used = [0]

    def ref(arr) -> Dict:
        a = np.asarray(arr, dtype="<f8")
        off = used[0]
        chunks.append(a.tobytes(order="C"))
        used[0] += a.size
        return {"offset": off, "shape": list(a.shape)}

    entries = []
    for nid in g.topo_order():
        node = g.nodes[nid]
        e: Dict = {"id": nid, "kind": node.kind}
        params = {p: getattr(node, p) for p in _PARAMS.get(node.kind, ())}
        if params:
            e["params"] = params
        if node.kind in _TENSORS:
            e["tensors"] = {f: ref(getattr(node, f)) for f in _TENSORS[node.kind]}
        elif node.kind == "polyact":
            e["tensors"] = {f"c{k}": ref(c) for k, c in enumerate(node.coeffs)}
        elif node.kind == "polyskip":
            e["tensors"] = {k: ref(node.coeffs[k]) for k in PS_KEYS}
        entries.append(e)
    doc = {
        "version": FORMAT_VERSION,
        "nodes": entries,
        "edges": [[s, d] for s, d in g.edges],
        "weights": base64.b64encode(b"".join(chunks)).decode("ascii"),
    }
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")


def load_model(path: str) -> ModelGraph:
    try:
        with open(path) as f:
            doc = json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise ModelFormatError(f"cannot read model file {path!r}: {e}") from e
    if not isinstance(doc, dict) or doc.get("version") != FORMAT_VERSION:
        raise ModelFormatError(
            f"unsupported model format version {doc.get('version') if isinstance(doc, dict) else None!r}")
    try:
        blob = np.frombuffer(base64.b64decode(doc["weights"]), dtype="<f8")
        g = ModelGraph()
        for e in doc["nodes"]:
            g.add(_node_from_entry(e, blob))
        for s, d in doc["edges"]:
            g.connect(s, d)
    except (KeyError, TypeError, ValueError) as e:
        raise ModelFormatError(f"malformed model file {path!r}: {e}") from e
    g.validate()
    return g


def load_model_views(path: str):
    """The neutral model as (graph, blob, specs): the base64 blob decoded
    once into a read-only float64 array, every node tensor a zero-copy view
    of it, specs[node id][field] = (offset, shape) of each tensor in the
    blob (polyact fields c0..cd, polyskip its monomial keys).  The loader
    behind lowering.load_lowered; same validation and errors as load_model."""
    try:
        with open(path) as f:
            doc = json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise ModelFormatError(f"cannot read model file {path!r}: {e}") from e
    if not isinstance(doc, dict) or doc.get("version") != FORMAT_VERSION:
        raise ModelFormatError(
            f"unsupported model format version {doc.get('version') if isinstance(doc, dict) else None!r}")
    specs: Dict[str, Dict[str, Tuple[int, Tuple[int, ...]]]] = {}
    try:
        blob = np.frombuffer(base64.b64decode(doc["weights"]), dtype="<f8")
        blob.flags.writeable = False
        g = ModelGraph()
        for e in doc["nodes"]:
            g.add(_node_from_entry(e, blob, views=True))
            specs[e["id"]] = {k: (int(v["offset"]), tuple(v["shape"])) for k, v in e.get("tensors", {}).items()}
        for s_, d_ in doc["edges"]:
            g.connect(s_, d_)
    except (KeyError, TypeError, ValueError) as e:
        raise ModelFormatError(f"malformed model file {path!r}: {e}") from e
    g.validate()
    return g, blob, specs


def _node_from_entry(e: Dict, blob: np.ndarray, views: bool = False) -> Node:
    kind = e["kind"]
    if kind not in TYPE_BY_KIND:
        raise ModelFormatError(f"unknown node kind {kind!r}")
    p = e.get("params", {})
    t = e.get("tensors", {})

    def tensor(name: str) -> np.ndarray:
        spec = t[name]
        shape = tuple(spec["shape"])
        n = int(np.prod(shape)) if shape else 1
        off = int(spec["offset"])
        if off < 0 or off + n > blob.size:
            raise ValueError(f"tensor {name!r} of node {e['id']!r} overruns the blob")
        v = blob[off:off + n].reshape(shape)
        return v if views else np.array(v, dtype=np.float64)

    nid = e["id"]
    if kind == "input":
        return InputNode(nid, p["channels"], p["height"], p["width"])
    if kind == "conv":
        return ConvNode(nid, tensor("weight"), tensor("bias"), p["stride"], p["padding"])
    if kind == "batchnorm":
        return BatchNormNode(nid, tensor("gamma"), tensor("beta"), tensor("mean"), tensor("std"))
    if kind == "polyact":
        return PolyActNode(nid, [tensor(f"c{k}") for k in range(len(t))])
    if kind == "polyskip":
        return PolySkipNode(nid, {k: tensor(k) for k in PS_KEYS})
    if kind == "avgpool":
        return AvgPoolNode(nid, p["k"], tensor("divisor"))
    if kind == "linear":
        return LinearNode(nid, tensor("weight"), tensor("bias"))
    if kind == "localpool":
        return LocalPoolNode(nid, p["k"], p["stride"], p["padding"], tensor("divisor"))
    if kind == "bipool":
        return BiPoolNode(nid, p["axis"], tensor("coeffs"))
    return TYPE_BY_KIND[kind](nid)
