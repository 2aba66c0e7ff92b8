"""Checkpoint ingest: a ResNet state dict -> ModelGraph -> the GPU path
(SURVEY.md section 8(f), row 4).

Restates the reference exporter's conversion (pkg/exporter/src/
levnet_exporter: checkpoint.py:11-47 readers, topology.py:36-112 layout,
exporting.py:77-194 key checks) on this package's graph types, so a trained
poly-ResNet can be fused, redistributed and run by the B200 kernels without
a round trip through the exporter CLI:

    g = graph_from_checkpoint("rn20.pt", "rn20")          # raw BN, as exported
    eng = engine_from_checkpoint("rn20.pt", "rn20")       # P2FR on the GPU, then Engine

Parameters stay raw (BN as gamma/beta/mean/std with std = sqrt(var + 1e-5),
exporting.py:23 and :161); no folding happens here -- fusing is the
pipeline's job (transforms.apply_pipeline).  Activation coefficients come
from the checkpoint (``<module>.coeffs``) or, for checkpoints without them,
from ``coeffs`` (the reference fits them with ``levnet fit-poly``, an
out-of-scope CLI).  Errors raise ExportError naming the offending key, with
the reference's wording.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .graph import (AddNode, AvgPoolNode, BatchNormNode, ConvNode, InputNode, LinearNode, ModelGraph, OutputNode,
                    PolyActNode, save_model)

BN_EPS = 1e-5  # exporting.py:23

# blocks per stage and native input resolution (topology.py:17-21)
VARIANTS = {
    "rn18": {"stages": (2, 2, 2, 2), "hw": 16},
    "rn20": {"stages": (3, 3, 3), "hw": 8},
    "rn32": {"stages": (5, 5, 5), "hw": 8},
}
BN_FIELDS = ("weight", "bias", "running_mean", "running_var")
IGNORED_SUFFIX = ".num_batches_tracked"


class ExportError(Exception):
    """Checkpoint cannot be converted; the message names the offending key
    (levnet_exporter errors.py)."""


def load_state_dict(path: str) -> Dict[str, np.ndarray]:
    """checkpoint.py:11-47: .npz archives, or torch.load of a bare state
    dict / a trainer checkpoint wrapping one under "state_dict"; every value
    as float64."""
    if str(path).endswith(".npz"):
        with np.load(path) as archive:
            raw = {k: archive[k] for k in archive.files}
    else:
        import torch
        try:
            obj = torch.load(path, map_location="cpu", weights_only=True)
        except Exception as e:  # noqa: BLE001 - the reader's own message
            raise ExportError(f"cannot read checkpoint {path!r}: {e}") from e
        if isinstance(obj, dict) and "state_dict" in obj and all(
                not torch.is_tensor(v) for k, v in obj.items() if k != "state_dict"):
            obj = obj["state_dict"]
        if not isinstance(obj, dict):
            raise ExportError(f"checkpoint {path!r} is not a state dict (got {type(obj).__name__})")
        raw = {k: v.detach().cpu().numpy() if torch.is_tensor(v) else v for k, v in obj.items()}
    state: Dict[str, np.ndarray] = {}
    for key, value in raw.items():
        arr = np.asarray(value)
        if arr.dtype == object or not np.issubdtype(arr.dtype, np.number):
            raise ExportError(f"checkpoint key {key!r} is not numeric")
        state[str(key)] = arr.astype(np.float64)
    return state


def infer_dims(state: Dict[str, np.ndarray]) -> Tuple[int, int, int]:
    """(base_width, in_channels, classes) from the stem and head (topology.py:134-153)."""
    for key in ("conv1.weight", "fc.weight"):
        if key not in state:
            raise ExportError(f"checkpoint is missing required key {key!r}")
    conv1, fc = state["conv1.weight"], state["fc.weight"]
    if conv1.ndim != 4:
        raise ExportError(f"checkpoint key 'conv1.weight' must be 4-D, got shape {tuple(conv1.shape)}")
    if fc.ndim != 2:
        raise ExportError(f"checkpoint key 'fc.weight' must be 2-D, got shape {tuple(fc.shape)}")
    return int(conv1.shape[0]), int(conv1.shape[1]), int(fc.shape[0])


@dataclass
class _Layer:
    """One learned plan node: graph id, state-dict module, kind, shape info."""
    id: str
    ckpt: str
    kind: str
    dims: Tuple[int, ...]  # conv: (cout, cin, k, stride, pad); bn / act: (C,); linear: (out, in)


def _plan(variant: str, width0: int, cin: int, classes: int, hw: int):
    """Node plan and edges of one variant (topology.py:36-112): a
    conv1/bn1/act1 stem, layer<s>.<b> basic blocks (downsample.0/.1 on the
    first block of every stage after the first), global pool, fc.  A join's
    first edge is the trunk, the second the skip."""
    if variant not in VARIANTS:
        raise ExportError(f"unknown variant {variant!r} (have {sorted(VARIANTS)})")
    spec = VARIANTS[variant]
    layers: List[_Layer] = []
    structural: List[Tuple[str, str]] = []  # (id, kind) of add / pool / output, in plan order
    edges: List[Tuple[str, str]] = []

    def chain(*ids):
        edges.extend(zip(ids, ids[1:]))

    def conv(i, ck, a, b, k, s, p):
        layers.append(_Layer(i, ck, "conv", (b, a, k, s, p)))
        return i

    def bn(i, ck, c):
        layers.append(_Layer(i, ck, "batchnorm", (c,)))
        return i

    def act(i, ck, c):
        layers.append(_Layer(i, ck, "polyact", (c,)))
        return i

    chain("in", conv("conv1", "conv1", cin, width0, 3, 1, 1), bn("bn1", "bn1", width0), act("act1", "act1", width0))
    tail, width = "act1", width0
    for si, blocks in enumerate(spec["stages"]):
        cout = width0 * 2 ** si
        for bi in range(blocks):
            name, pre = f"s{si + 1}b{bi + 1}", f"layer{si + 1}.{bi}"
            first = bi == 0 and si > 0
            chain(tail, conv(f"{name}.conva", f"{pre}.conv1", width, cout, 3, 2 if first else 1, 1),
                  bn(f"{name}.bna", f"{pre}.bn1", cout), act(f"{name}.acta", f"{pre}.act1", cout),
                  conv(f"{name}.convb", f"{pre}.conv2", cout, cout, 3, 1, 1), bn(f"{name}.bnb", f"{pre}.bn2", cout))
            join = f"{name}.join"
            structural.append((join, "add"))
            edges.append((f"{name}.bnb", join))
            if first:
                chain(tail, conv(f"{name}.convd", f"{pre}.downsample.0", width, cout, 1, 2, 0),
                      bn(f"{name}.bnd", f"{pre}.downsample.1", cout))
                edges.append((f"{name}.bnd", join))
            else:
                edges.append((tail, join))
            chain(join, act(f"{name}.actj", f"{pre}.act2", cout))
            tail, width = f"{name}.actj", cout
    hw_out = hw // 2 ** (len(spec["stages"]) - 1)
    if hw_out < 1:
        raise ExportError(f"input size {hw} collapses below 1x1 for {variant}")
    layers.append(_Layer("fc", "fc", "linear", (classes, width)))
    chain(tail, "pool", "fc", "out")
    return layers, structural, edges, hw_out * hw_out


def _expected(layer: _Layer) -> Dict[str, Tuple[Optional[Tuple[int, ...]], bool]]:
    """State-dict keys of one learned node: key -> (shape or None, required) (topology.py:115-131)."""
    k = layer.ckpt
    if layer.kind == "conv":
        cout, cin, ks = layer.dims[:3]
        return {f"{k}.weight": ((cout, cin, ks, ks), True), f"{k}.bias": ((cout,), False)}
    if layer.kind == "batchnorm":
        return {f"{k}.{f}": (layer.dims, True) for f in BN_FIELDS}
    if layer.kind == "polyact":
        return {f"{k}.coeffs": (None, False)}
    return {f"{k}.weight": (layer.dims, True), f"{k}.bias": ((layer.dims[0],), True)}


def graph_from_state(state: Dict[str, np.ndarray], variant: str, *, coeffs: Optional[Sequence[float]] = None,
                     input_hw: Optional[int] = None) -> ModelGraph:
    """exporting.py:77-186 on ModelGraph: check every key against the
    variant's layout (missing / wrong shape / unmapped key -> ExportError
    naming it), then build the raw graph."""
    width0, cin, classes = infer_dims(state)
    hw = input_hw or VARIANTS.get(variant, {"hw": 8})["hw"]
    layers, structural, edges, pool_k = _plan(variant, width0, cin, classes, hw)
    consumed = set()
    for layer in layers:
        for key, (shape, required) in _expected(layer).items():
            if key not in state:
                if required:
                    raise ExportError(f"checkpoint is missing required key {key!r}")
                continue
            got = state[key].shape
            if shape is None:
                if state[key].ndim != 1 or got[0] < 2:
                    raise ExportError(f"checkpoint key {key!r} must be a coefficient vector (c0..cd), "
                                      f"got shape {tuple(got)}")
            elif got != shape:
                raise ExportError(f"checkpoint key {key!r} has shape {tuple(got)}, expected {shape}")
            consumed.add(key)
    for key in sorted(state):
        if key not in consumed and not key.endswith(IGNORED_SUFFIX):
            raise ExportError(f"checkpoint key {key!r} does not map to any {variant} layer")
    act_keys = [f"{l.ckpt}.coeffs" for l in layers if l.kind == "polyact"]
    embedded = [k for k in act_keys if k in state]
    if embedded and len(embedded) != len(act_keys):
        missing = next(k for k in act_keys if k not in state)
        raise ExportError(f"checkpoint embeds activation coefficients for {len(embedded)} of {len(act_keys)} "
                          f"activations; {missing!r} is missing")
    if embedded:
        if len({state[k].shape[0] for k in act_keys}) != 1:
            raise ExportError(f"embedded activation coefficient vectors disagree on length: "
                              f"{sorted({state[k].shape[0] for k in act_keys})}")
        coeffs_of = {k: state[k] for k in act_keys}
    else:
        if coeffs is None:
            raise ExportError("checkpoint has no activation coefficients; pass coeffs (c0..cd), "
                              "e.g. from levnet fit-poly")
        shared = np.asarray(coeffs, dtype=np.float64)
        if shared.ndim != 1 or shared.shape[0] < 2:
            raise ExportError(f"coeffs must be a coefficient vector (c0..cd), got shape {tuple(shared.shape)}")
        coeffs_of = {k: shared for k in act_keys}

    g = ModelGraph()
    g.add(InputNode("in", channels=cin, height=hw, width=hw))
    for layer in layers:
        k = layer.ckpt
        if layer.kind == "conv":
            cout, _, _, stride, pad = layer.dims
            g.add(ConvNode(layer.id, weight=state[f"{k}.weight"].copy(),
                           bias=state.get(f"{k}.bias", np.zeros(cout)).copy(), stride=stride, padding=pad))
        elif layer.kind == "batchnorm":
            var = state[f"{k}.running_var"]
            if not np.all(var + BN_EPS > 0):
                raise ExportError(f"checkpoint key '{k}.running_var' has entries <= {-BN_EPS}; "
                                  f"cannot form a positive sigma")
            g.add(BatchNormNode(layer.id, gamma=state[f"{k}.weight"].copy(), beta=state[f"{k}.bias"].copy(),
                                mean=state[f"{k}.running_mean"].copy(), std=np.sqrt(var + BN_EPS)))
        elif layer.kind == "polyact":
            g.add(PolyActNode(layer.id, coeffs=[np.asarray(float(c)) for c in coeffs_of[f"{k}.coeffs"]]))
        else:
            g.add(LinearNode(layer.id, weight=state[f"{k}.weight"].copy(), bias=state[f"{k}.bias"].copy()))
    for nid, kind in structural:
        g.add(AddNode(nid))
    g.add(AvgPoolNode("pool", k=pool_k, divisor=np.asarray(1.0 / pool_k)))
    g.add(OutputNode("out"))
    for s, d in edges:
        g.connect(s, d)
    g.validate()
    return g


def graph_from_checkpoint(path: str, variant: str, **kw) -> ModelGraph:
    """load_state_dict + graph_from_state (exporting.py:189-194)."""
    return graph_from_state(load_state_dict(path), variant, **kw)


def export_state(state: Dict[str, np.ndarray], variant: str, out: str, **kw) -> str:
    """Write the converted graph in the neutral JSON format; returns the
    sha256 of the weight blob (the exporter manifest's weight_hash)."""
    g = graph_from_state(state, variant, **kw)
    save_model(g, out)
    import base64
    import json
    with open(out) as f:
        return hashlib.sha256(base64.b64decode(json.load(f)["weights"])).hexdigest()


def engine_from_checkpoint(path: str, variant: str, strategy: str = "P2FR", **kw):
    """Checkpoint -> raw graph -> apply_pipeline(strategy) (fusing on the
    host, the channelwise redistribution on the GPU) -> a resident Engine.
    Returns (engine, redistributed graph, pass report)."""
    from .runtime import Engine
    from .transforms import apply_pipeline
    g = graph_from_checkpoint(path, variant, **kw)
    rg, report = apply_pipeline(g, strategy)
    return Engine(rg), rg, report
