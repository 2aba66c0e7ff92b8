"""Lower a ModelGraph to the flat tables libpcnn executes.

Three products:

* the float64 **master** parameter layout -- every node's tensors in the
  device-friendly padded form the kernels and the redistribution kernel
  index directly (conv weights [Npad][Kp] with K ordered (channel block, ky,
  kx, channel-in-block); per-channel vectors padded to the tensor's blocked
  width; scalars broadcast per channel);
* the **units**: fused kernels.  A conv absorbs, when each intermediate value
  has a single consumer, a following batchnorm, a residual add or quadratic
  join with its skip tensor, a polynomial activation, and a 2x2 sum pool, a
  2x2 pairwise bivariate pool, or the global pool.  A dense layer absorbs a
  preceding flatten or global pool and a following activation.  Everything
  else becomes a standalone kernel, so any graph the IR accepts runs on the
  GPU;
* the **pack** ops turning the float64 master into the float32 images the
  units read (plus the tcgen05 hi/lo weight images).

This is host bookkeeping (the reference re-walks its graph per image,
graph.py:413-426); no numerics happen here except layout permutation.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple


import numpy as np

from . import _lib as L
from .graph import (load_model_views, AddNode, AvgPoolNode, BatchNormNode, BiPoolNode, ConvNode, FlattenNode,
                    GraphError, InputNode, LinearNode, LocalPoolNode, ModelGraph, OutputNode,
                    PolyActNode, PolySkipNode, PS_KEYS)

ALIGN = 256  # floats


def cb_for(c: int) -> int:
    """Channel block of a tensor with c channels."""
    if c % 32 == 0:
        return 32
    for cb in (4, 8, 16):
        if c <= cb:
            return cb
    return 32


def cpad_for(c: int) -> int:
    cb = cb_for(c)
    return (c + cb - 1) // cb * cb


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


@dataclass
class Tensor:
    c: int
    h: int
    w: int
    is_vector: bool
    offset: int = 0  # floats per batch-element multiple (see Lowered.tensor_descs)

    @property
    def cb(self) -> int:
        return cb_for(self.c)

    @property
    def nblk(self) -> int:
        return cpad_for(self.c) // self.cb

    @property
    def cpad(self) -> int:
        return cpad_for(self.c)

    def floats(self, batch: int) -> int:
        """Workspace floats: the larger of the float32 blocked layout and the
        split fp16 hi/lo layout (two planes [C/8][B][H+2][W+2][8] halves) --
        libpcnn picks the format per tensor (csrc/common.cuh)."""
        fp32 = batch * self.cpad * self.h * self.w
        if self.is_vector:
            return fp32
        # (the parity layout of stride-2 inputs rounds the padded grid up to even)
        return max(fp32, -(-self.cpad // 8) * 8 * batch * ((self.h + 3) // 2 * 2) * ((self.w + 3) // 2 * 2))


@dataclass
class Slot:
    """One tensor of one node in the float64 master."""
    offset: int
    n: int
    meta: Dict = field(default_factory=dict)


@dataclass
class Lowered:
    graph: ModelGraph
    shapes: Dict[str, Tuple[int, ...]]
    tensors: List[Tensor]
    units: List[Dict]
    unit_nodes: List[List[str]]
    slots: Dict[str, Dict[str, Slot]]
    master_size: int
    pack_ops: List[Tuple]
    packed_size: int
    input_tensor: int
    output_tensor: int
    out_shape: Tuple[int, ...]
    scalar: Dict[Tuple[str, str], bool]

    # -- descriptor tables for the C ABI --------------------------------------
    def tensor_descs(self, batch: int, scale_log2=None):
        descs = []
        off = 0
        for i, t in enumerate(self.tensors):
            descs.append(L.TensorDesc(c=t.c, h=t.h, w=t.w, cb=t.cb, nblk=t.nblk,
                                      is_vector=int(t.is_vector), offset=off,
                                      scale_log2=int(scale_log2[i]) if scale_log2 is not None else 0))
            off += _align(t.floats(batch))
        return L.array(L.TensorDesc, descs), off

    def unit_descs(self, impl: int = 0):
        out = []
        for u in self.units:
            d = dict(u)
            if d.get("kind") == L.UNIT_CONV and impl:
                d["impl"] = impl
            out.append(L.UnitDesc(**d))
        return L.array(L.UnitDesc, out)

    def pack_descs(self):
        return L.array(L.PackDesc, [L.PackDesc(kind=op[0], src=op[1], dst=op[2], n=op[3], rows=op[4], k=op[5],
                                               aux=op[6] if len(op) > 6 else 0,
                                               reserved=op[7] if len(op) > 7 else 0)
                                    for op in self.pack_ops])


# ---------------------------------------------------------------------------
# master layout: upload / download
# ---------------------------------------------------------------------------

def _vec(arr, cpad: int) -> np.ndarray:
    a = np.asarray(arr, dtype=np.float64)
    out = np.zeros(cpad)
    if a.ndim == 0:
        out[:] = float(a)
    else:
        out[:a.shape[0]] = a
    return out


def conv_weight_to_master(w: np.ndarray, npad: int, cin: int) -> Tuple[np.ndarray, Dict]:
    o, i, kh, kw = w.shape
    cb = cb_for(cin)
    nblk = cpad_for(cin) // cb
    full = np.zeros((npad, nblk * cb, kh, kw))
    full[:o, :i] = w
    # [Npad][nblk][cb][kh][kw] -> [Npad][nblk][kh][kw][cb]
    m = full.reshape(npad, nblk, cb, kh, kw).transpose(0, 1, 3, 4, 2).reshape(npad, -1)
    return m, {"o": o, "i": i, "kh": kh, "kw": kw, "cb": cb, "nblk": nblk, "npad": npad,
               "kp": nblk * kh * kw * cb}


def conv_weight_from_master(m: np.ndarray, meta: Dict) -> np.ndarray:
    npad, nblk, cb, kh, kw = meta["npad"], meta["nblk"], meta["cb"], meta["kh"], meta["kw"]
    full = m.reshape(npad, nblk, kh, kw, cb).transpose(0, 1, 4, 2, 3).reshape(npad, nblk * cb, kh, kw)
    if "s2d" in meta:
        return s2d_weight_back(full[:meta["o"]], meta["s2d"])
    return np.array(full[:meta["o"], :meta["i"]])


# ---------------------------------------------------------------------------
# space-to-depth stem: a k x k / stride-2 conv (pad p, odd k) on a cin <= 4
# image is the same function as a k' x k' / stride-1 conv on the image cut
# into 2 x 2 blocks, X'[(dy,dx,c)][i][j] = X[c][2i+dy][2j+dx]:
# W'[o][(dy,dx,c)][ti][tj] = W[o][c][2(ti-P)+p+dy][2(tj-P)+p+dx] (0 outside the
# kernel), taps reaching P blocks back.  For 7x7/s2/p3: k' = 4, P = 2.  The
# ingest stores X' shifted by one block (a zero first row and column, H/2+1 x
# W/2+1), which turns the (-2..+1) reach into an ordinary pad-1 conv that
# yields exactly H/2 x W/2 outputs: 4 cin <= 16 channels feed the halo-tile
# kernel (one 16-channel chunk, 16 taps) instead of a 49-tap gather.
# ---------------------------------------------------------------------------

S2D_K, S2D_P = 4, 2  # the 7x7 / s2 / p3 stem


def s2d_eligible(g: ModelGraph, shapes, nid: str) -> bool:
    node = g.nodes[nid]
    if not isinstance(node, ConvNode) or node.stride != 2 or node.padding != 3:
        return False
    o, i, kh, kw = node.weight.shape
    if kh != 7 or kw != 7 or i > 4:
        return False
    preds = [s for s, d in g.edges if d == nid]
    if len(preds) != 1 or not isinstance(g.nodes[preds[0]], InputNode):
        return False
    if len(g.consumer_edges(preds[0])) != 1:
        return False
    c, h, w = shapes[preds[0]]
    return h % 2 == 0 and w % 2 == 0


def s2d_weight(w: np.ndarray) -> np.ndarray:
    o, cin, k, _ = w.shape
    p = (k - 1) // 2
    out = np.zeros((o, 4 * cin, S2D_K, S2D_K))
    for ti in range(S2D_K):
        for dy in range(2):
            ky = 2 * (ti - S2D_P) + p + dy
            if not 0 <= ky < k:
                continue
            for tj in range(S2D_K):
                for dx in range(2):
                    kx = 2 * (tj - S2D_P) + p + dx
                    if not 0 <= kx < k:
                        continue
                    c0 = (dy * 2 + dx) * cin
                    out[:, c0:c0 + cin, ti, tj] = w[:, :, ky, kx]
    return out


def s2d_weight_back(w2: np.ndarray, info: Dict) -> np.ndarray:
    o, cin, k = w2.shape[0], info["cin"], info["k"]
    p = (k - 1) // 2
    w = np.zeros((o, cin, k, k))
    for ky in range(k):
        dy, ti = (ky - p) % 2, (ky - p - (ky - p) % 2) // 2 + S2D_P
        for kx in range(k):
            dx, tj = (kx - p) % 2, (kx - p - (kx - p) % 2) // 2 + S2D_P
            c0 = (dy * 2 + dx) * cin
            w[:, :, ky, kx] = w2[:, c0:c0 + cin, ti, tj]
    return w


def build_master(g: ModelGraph, shapes, get=None) -> Tuple[Dict[str, Dict[str, Slot]], List[np.ndarray], int, Dict]:
    """Assign master offsets for every parameter and return the float64 chunks.

    get(node, field) supplies a parameter tensor (default: the node's own
    attribute; polyact fields are c0..cd, polyskip fields its monomial keys).
    load_lowered passes encoded blob indices instead of values, so the same
    layout code yields the index map of the neutral-format loader."""
    if get is None:
        def get(node, field):
            if isinstance(node, PolyActNode):
                return node.coeffs[int(field[1:])]
            if isinstance(node, PolySkipNode):
                return node.coeffs[field]
            return getattr(node, field)
    slots: Dict[str, Dict[str, Slot]] = {}
    chunks: List[Tuple[int, np.ndarray]] = []
    scalar: Dict[Tuple[str, str], bool] = {}
    pos = [0]

    def put(nid: str, name: str, arr: np.ndarray, **meta) -> None:
        arr = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1)
        off = pos[0]
        chunks.append((off, arr))
        pos[0] = off + _align(arr.size)
        slots.setdefault(nid, {})[name] = Slot(off, arr.size, meta)

    preds: Dict[str, List[str]] = {nid: [] for nid in g.nodes}
    for s, d in g.edges:
        preds[d].append(s)
    for nid in g.topo_order():
        node = g.nodes[nid]
        c_out = shapes[nid][0]
        cp = cpad_for(c_out)
        if isinstance(node, ConvNode):
            cin = shapes[preds[nid][0]][0]
            w = get(node, "weight")
            if s2d_eligible(g, shapes, nid):
                m, meta = conv_weight_to_master(s2d_weight(w), cp, 4 * cin)
                meta["s2d"] = {"cin": cin, "k": w.shape[2]}
                meta["i"] = cin
            else:
                m, meta = conv_weight_to_master(w, cp, cin)
            put(nid, "weight", m, **meta)
            put(nid, "bias", _vec(get(node, "bias"), cp))
        elif isinstance(node, LinearNode):
            w = get(node, "weight")
            k, n = w.shape
            put(nid, "weight", w, k=k, n=n)
            put(nid, "bias", _vec(get(node, "bias"), cp))
        elif isinstance(node, BatchNormNode):
            std = np.ones(cp)
            std[:c_out] = get(node, "std")
            put(nid, "bn", np.concatenate([_vec(get(node, "gamma"), cp), _vec(get(node, "beta"), cp),
                                           _vec(get(node, "mean"), cp), std]), cpad=cp, c=c_out)
        elif isinstance(node, PolyActNode):
            cs = [get(node, f"c{i}") for i in range(node.degree + 1)]
            put(nid, "coeffs", np.concatenate([_vec(c, cp) for c in cs]),
                cpad=cp, c=c_out, deg=node.degree)
            for i, c in enumerate(cs):
                scalar[(nid, f"c{i}")] = np.asarray(c).ndim == 0
        elif isinstance(node, PolySkipNode):
            cs = {k: get(node, k) for k in PS_KEYS}
            put(nid, "coeffs", np.concatenate([_vec(cs[k], cp) for k in PS_KEYS]),
                cpad=cp, c=c_out)
            for k in PS_KEYS:
                scalar[(nid, k)] = np.asarray(cs[k]).ndim == 0
        elif isinstance(node, (AvgPoolNode, LocalPoolNode)):
            dv = get(node, "divisor")
            put(nid, "divisor", np.asarray([float(dv)]))
            scalar[(nid, "divisor")] = np.asarray(dv).ndim == 0
        elif isinstance(node, BiPoolNode):
            c = np.asarray(get(node, "coeffs"), dtype=np.float64)
            d = c.shape[0] - 1
            flat = [_vec(c[i, j], cp) for i in range(d + 1) for j in range(d + 1)]
            put(nid, "coeffs", np.concatenate(flat), cpad=cp, c=c_out, deg=d)
            scalar[(nid, "coeffs")] = c.ndim == 2
    return slots, chunks, pos[0], scalar


def master_array(chunks, size: int) -> np.ndarray:
    m = np.zeros(size)
    for off, arr in chunks:
        m[off:off + arr.size] = arr
    return m


def graph_from_master(lw: "Lowered", master: np.ndarray, vector_keys=(), scalar_keys=None) -> ModelGraph:
    """Rebuild a ModelGraph (copy of lw.graph) from a float64 master array.

    Coefficient shapes follow the reference: a coefficient that was a
    scalar stays one, except the (node, key) pairs in ``vector_keys``, which
    come back per-channel; pairs in ``scalar_keys`` come back as scalars.
    The default ``scalar_keys`` are the leading terms the channelwise pass
    pins to constants (transforms.py:689, :695-697).
    """
    g = lw.graph.copy()
    shapes = lw.shapes
    vector_keys = set(vector_keys)
    scalar_keys = set(scalar_keys or ())

    def shape_of(nid, key, v):
        if (nid, key) in scalar_keys:
            return np.asarray(v[0])
        if (nid, key) in vector_keys or not lw.scalar.get((nid, key), False):
            return np.array(v)
        return np.asarray(v[0])

    for nid, sl in lw.slots.items():
        node = g.nodes[nid]
        c_out = shapes[nid][0]

        def get(name):
            s = sl[name]
            return master[s.offset:s.offset + s.n]

        if isinstance(node, ConvNode):
            node.weight = conv_weight_from_master(get("weight"), sl["weight"].meta)
            node.bias = np.array(get("bias")[:node.weight.shape[0]])
        elif isinstance(node, LinearNode):
            k, n = sl["weight"].meta["k"], sl["weight"].meta["n"]
            node.weight = np.array(get("weight").reshape(k, n))
            node.bias = np.array(get("bias")[:k])
        elif isinstance(node, BatchNormNode):
            cp = sl["bn"].meta["cpad"]
            v = get("bn").reshape(4, cp)[:, :c_out]
            node.gamma, node.beta, node.mean, node.std = (np.array(v[i]) for i in range(4))
        elif isinstance(node, PolyActNode):
            cp = sl["coeffs"].meta["cpad"]
            v = get("coeffs").reshape(-1, cp)[:, :c_out]
            node.coeffs = [shape_of(nid, f"c{i}", v[i]) for i in range(v.shape[0])]
        elif isinstance(node, PolySkipNode):
            cp = sl["coeffs"].meta["cpad"]
            v = get("coeffs").reshape(6, cp)[:, :c_out]
            node.coeffs = {k: shape_of(nid, k, v[i]) for i, k in enumerate(PS_KEYS)}
        elif isinstance(node, (AvgPoolNode, LocalPoolNode)):
            node.divisor = np.asarray(get("divisor")[0])
        elif isinstance(node, BiPoolNode):
            cp = sl["coeffs"].meta["cpad"]
            d = sl["coeffs"].meta["deg"]
            v = get("coeffs").reshape(d + 1, d + 1, cp)[:, :, :c_out]
            node.coeffs = np.array(v[:, :, 0]) if lw.scalar[(nid, "coeffs")] else np.array(v)
    return g


# ---------------------------------------------------------------------------
# units
# ---------------------------------------------------------------------------

class _Builder:
    def __init__(self, g: ModelGraph, slots, master_size: int, use_tc: bool):
        self.g = g
        self.shapes = g.validate()
        self.slots = slots
        self.tensors: List[Tensor] = []
        self.units: List[Dict] = []
        self.unit_nodes: List[List[str]] = []
        self.value: Dict[str, int] = {}
        self.fused: set = set()
        self.pack: List[Tuple] = []
        self.packed = 0
        self.use_tc = use_tc
        self.preds: Dict[str, List[str]] = {nid: [] for nid in g.nodes}
        for s, d in g.edges:
            self.preds[d].append(s)

    # -- helpers -------------------------------------------------------------
    def tensor(self, shape) -> int:
        if len(shape) == 3:
            self.tensors.append(Tensor(shape[0], shape[1], shape[2], False))
        else:
            self.tensors.append(Tensor(shape[0], 1, 1, True))
        return len(self.tensors) - 1

    def single(self, nid: str) -> Optional[Tuple[str, int]]:
        edges = self.g.consumer_edges(nid)
        return edges[0] if len(edges) == 1 else None

    def cast(self, nid: str, name: str, sub: int = 0, n: Optional[int] = None) -> int:
        s = self.slots[nid][name]
        n = s.n - sub if n is None else n
        dst = self.packed
        self.pack.append((L.PACK_CAST, s.offset + sub, dst, n, 0, 0))
        self.packed += _align(n)
        return dst

    def cast_pair(self, a: str, b: str) -> int:
        """Two bivariate coefficient sets back to back (BI2 epilogue)."""
        sa, sb = self.slots[a]["coeffs"], self.slots[b]["coeffs"]
        dst = self.packed
        self.pack.append((L.PACK_CAST, sa.offset, dst, sa.n, 0, 0))
        self.pack.append((L.PACK_CAST, sb.offset, dst + sa.n, sb.n, 0, 0))
        self.packed += _align(sa.n + sb.n)
        return dst

    def affine(self, nid: str) -> int:
        s = self.slots[nid]["bn"]
        cp = s.meta["cpad"]
        dst = self.packed
        self.pack.append((L.PACK_BN_AFFINE, s.offset, dst, cp, 0, 0))
        self.packed += _align(2 * cp)
        return dst

    def tc_image(self, nid: str) -> int:
        s = self.slots[nid]["weight"]
        npad, kp = s.meta["npad"], s.meta["kp"]
        ntile = npad if npad <= 128 else 128
        kb = (kp + 31) // 32
        floats = ((npad + ntile - 1) // ntile) * kb * 2 * ntile * 32
        dst = self.packed
        self.pack.append((L.PACK_TC_WEIGHTS, s.offset, dst, floats, npad, kp))
        self.packed += _align(floats)
        return dst

    def tc16_image(self, nid: str) -> Tuple[int, int]:
        """fp16x2 image (64 fp16 per 128-byte row, one float per element for
        hi+lo) and its {max|w|, 2^-e} scale pair."""
        s = self.slots[nid]["weight"]
        npad, kp = s.meta["npad"], s.meta["kp"]
        ntile = npad if npad <= 128 else 128
        kb = (kp + 63) // 64
        floats = ((npad + ntile - 1) // ntile) * kb * ntile * 64
        dst = self.packed
        self.packed += _align(floats)
        scale = self.packed
        self.packed += _align(2)
        self.pack.append((L.PACK_TC16_WEIGHTS, s.offset, dst, floats, npad, kp, scale))
        return dst, scale

    def tcss_image(self, nid: str, scale: int) -> int:
        """fp16x2 image of the shared-memory (halo tile) kernel: blocks of
        [2 x 8-channel groups][hi NT rows | lo NT rows][8] per (16-channel
        chunk, tap); shares the fp16x2 image's scale pair."""
        s = self.slots[nid]["weight"]
        m = s.meta
        npad, kp, taps, cb = m["npad"], m["kp"], m["kh"] * m["kw"], m["cb"]
        ntile = npad if npad <= 128 else 128
        cpad = kp // taps
        floats = ((npad + ntile - 1) // ntile) * (-(-cpad // 16)) * taps * 16 * ntile
        dst = self.packed
        self.packed += _align(floats)
        self.pack.append((L.PACK_TCSS_WEIGHTS, s.offset, dst, floats, npad, kp, scale, taps | (cb << 16)))
        return dst

    def emit(self, nodes: List[str], **u) -> None:
        self.units.append(u)
        self.unit_nodes.append(nodes)

    # -- lowering -------------------------------------------------------------
    def run(self):
        g = self.g
        order = g.topo_order()
        in_id, out_id = g.input_id(), g.output_id()
        for nid in order:
            if nid in self.fused:
                continue
            node = g.nodes[nid]
            if isinstance(node, InputNode):
                c, h, w = self.shapes[nid]
                nxt = self.single(nid)
                s2d = nxt is not None and "s2d" in self.slots.get(nxt[0], {}).get("weight", Slot(0, 0, {})).meta
                # space-to-depth stem: the ingest writes the image as 2x2 blocks
                # behind a zero first row and column
                t = self.tensor((4 * c, h // 2 + 1, w // 2 + 1) if s2d else (c, h, w))
                self.value[nid] = t
                self.input_tensor = t
                self.emit([nid], kind=L.UNIT_INGEST, out=t, flags=L.FLAG_S2D if s2d else 0)
            elif isinstance(node, ConvNode):
                self.lower_conv(nid)
            elif isinstance(node, LinearNode):
                self.lower_linear(nid)
            elif isinstance(node, OutputNode):
                src = self.value[self.preds[nid][0]]
                self.output_tensor = src
                self.emit([nid], kind=L.UNIT_COPYOUT, in_=src)
            elif isinstance(node, FlattenNode):
                nxt = self.single(nid)
                if nxt and isinstance(g.nodes[nxt[0]], LinearNode):
                    self.fused.add(nid)  # read by the dense layer directly
                    continue
                t = self.tensor(self.shapes[nid])
                self.emit([nid], kind=L.UNIT_FLATTEN, in_=self.value[self.preds[nid][0]], out=t)
                self.value[nid] = t
            elif isinstance(node, AvgPoolNode):
                nxt = self.single(nid)
                if nxt and isinstance(g.nodes[nxt[0]], LinearNode):
                    self.fused.add(nid)
                    continue
                t = self.tensor(self.shapes[nid])
                self.emit([nid], kind=L.UNIT_GLOBALPOOL, in_=self.value[self.preds[nid][0]], out=t,
                          pool_off=self.cast(nid, "divisor"))
                self.value[nid] = t
            else:
                self.lower_eltwise(nid)
        self.output_shape = self.shapes[self.preds[out_id][0]]
        return self

    def lower_conv(self, nid: str):
        g, sh = self.g, self.shapes
        node = g.nodes[nid]
        src = self.value[self.preds[nid][0]]
        wmeta = self.slots[nid]["weight"].meta
        u = dict(kind=L.UNIT_CONV, in_=src, cin=wmeta["i"], cout=wmeta["o"], kh=wmeta["kh"], kw=wmeta["kw"],
                 stride=node.stride, pad=node.padding, npad=wmeta["npad"])
        if "s2d" in wmeta:
            # 4x4 / stride-1 / pad-1 conv over the shifted blocked image
            u.update(cin=4 * wmeta["i"], stride=1, pad=1)
        u["w_off"] = self.cast(nid, "weight")
        u["b_off"] = self.cast(nid, "bias")
        chain = [nid]
        cur = nid
        nxt = self.single(cur)
        if nxt and isinstance(g.nodes[nxt[0]], BatchNormNode):
            cur = nxt[0]
            chain.append(cur)
            u["affine_off"] = self.affine(cur)
            nxt = self.single(cur)
        if nxt and isinstance(g.nodes[nxt[0]], (AddNode, PolySkipNode)):
            join, pos = nxt
            other = [p for i, p in enumerate(self.preds[join]) if i != pos][0]
            if other in self.value and other not in chain:
                u["in2"] = self.value[other]
                if isinstance(g.nodes[join], AddNode):
                    u["residual"] = 1
                else:
                    u["residual"] = 2 if pos == 0 else 3
                    u["res_off"] = self.cast(join, "coeffs")
                cur = join
                chain.append(cur)
                nxt = self.single(cur)
            elif other not in self.value:
                # the skip branch is computed later: postpone the join to it
                nxt = None
        if nxt and isinstance(g.nodes[nxt[0]], PolyActNode) and not isinstance(g.nodes[cur], PolySkipNode):
            cur = nxt[0]
            chain.append(cur)
            u["poly_deg"] = g.nodes[cur].degree
            u["poly_off"] = self.cast(cur, "coeffs")
            nxt = self.single(cur)
        out_shape = sh[cur]
        k, st, pd = wmeta["kh"], u["stride"], u["pad"]
        # shapes the halo-tile kernel (conv_ss) runs; it has no 2x2-window
        # epilogue, so for these a following 2x2 pool stays a separate unit
        # (measured: conv_ss + pool pass beats the TMEM-A kernel with the
        # pool fused, VGG-11; PCNN_FUSE_WINDOW_POOL=1 restores the fusion)
        ss_shape = (self.use_tc and wmeta["npad"] % 16 == 0 and wmeta["npad"] >= 16
                    and wmeta["kh"] == wmeta["kw"] and st in (1, 2)
                    and ((k == 3 and pd == 1) or (k == 1 and pd == 0) or (k == S2D_K and pd == 1 and st == 1))
                    and ((cp := wmeta["kp"] // (k * k)) in (4, 8) or cp % 16 == 0))
        window_ok = not ss_shape
        # band epilogue of the halo-tile kernel (conv_ss.cu band_pool): a
        # following local pool or 2x2 bivariate pool computed over row bands
        # in the conv's epilogue when the conv is stride 1, has >= 32 output
        # channels and its grid rows (input width + 1) fit a 128-row tile
        # (and are >= 9 long: tiny maps keep whole tiles / stream-K and a
        # separate pool pass)
        band_ok = (ss_shape and st == 1 and wmeta["npad"] >= 32 and not u.get("residual")
                   and 8 <= self.tensors[src].w and self.tensors[src].w + 1 <= 128)
        post_pool = None  # (first, second) BiPool nodes lowered as one 2x2 pool unit after the conv
        if nxt:
            pn = g.nodes[nxt[0]]
            nn = self.single(nxt[0]) if isinstance(pn, BiPoolNode) else None
            bi_pair = (nn is not None and isinstance(g.nodes[nn[0]], BiPoolNode) and g.nodes[nn[0]].axis != pn.axis
                       and g.nodes[nn[0]].degree == pn.degree and pn.degree <= 4)
            if band_ok and isinstance(pn, LocalPoolNode) and pn.k <= 2 * pn.stride + 1 and pn.padding < pn.k:
                cur = nxt[0]
                chain.append(cur)
                u["pool"] = L.POOL_LOCAL
                u["pool_geom"] = pn.k | (pn.stride << 8) | (pn.padding << 16)
                u["pool_off"] = self.cast(cur, "divisor")
                out_shape = sh[cur]
            elif band_ok and bi_pair:
                chain += [nxt[0], nn[0]]
                cur = nn[0]
                u["pool"] = L.POOL_BI2
                u["pool_deg"] = pn.degree
                u["pool_order"] = 0 if pn.axis == "w" else 1
                u["pool_off"] = self.cast_pair(nxt[0], nn[0])
                out_shape = sh[cur]
            elif not window_ok and isinstance(pn, (LocalPoolNode, BiPoolNode)):
                nn = self.single(nxt[0]) if isinstance(pn, BiPoolNode) else None
                if nn and isinstance(g.nodes[nn[0]], BiPoolNode) and g.nodes[nn[0]].axis != pn.axis \
                        and g.nodes[nn[0]].degree == pn.degree and pn.degree <= 4:
                    post_pool = (nxt[0], nn[0])
            elif isinstance(pn, LocalPoolNode) and pn.k == 2 and pn.stride == 2 and pn.padding == 0:
                cur = nxt[0]
                chain.append(cur)
                u["pool"] = L.POOL_SUM2
                u["pool_off"] = self.cast(cur, "divisor")
                out_shape = sh[cur]
            elif isinstance(pn, BiPoolNode):
                nn = self.single(nxt[0])
                if nn and isinstance(g.nodes[nn[0]], BiPoolNode) and g.nodes[nn[0]].axis != pn.axis \
                        and g.nodes[nn[0]].degree == pn.degree and pn.degree <= 4:
                    chain += [nxt[0], nn[0]]
                    cur = nn[0]
                    u["pool"] = L.POOL_BI2
                    u["pool_deg"] = pn.degree
                    u["pool_order"] = 0 if pn.axis == "w" else 1
                    u["pool_off"] = self.cast_pair(nxt[0], nn[0])
                    out_shape = sh[cur]
            elif isinstance(pn, AvgPoolNode):
                cur = nxt[0]
                chain.append(cur)
                u["pool"] = L.POOL_GLOBAL
                u["pool_off"] = self.cast(cur, "divisor")
                out_shape = sh[cur]
        if self.use_tc and wmeta["npad"] % 16 == 0 and wmeta["npad"] >= 16:
            u["tc_off"] = self.tc_image(nid)
            u["tc16_off"], u["tc16_scale_off"] = self.tc16_image(nid)
            if ss_shape and u.get("pool", 0) in (L.POOL_NONE, L.POOL_GLOBAL, L.POOL_LOCAL, L.POOL_BI2):
                u["tcss_off"] = self.tcss_image(nid, u["tc16_scale_off"])
        t = self.tensor(out_shape)
        u["out"] = t
        for c in chain[1:]:
            self.fused.add(c)
        self.value[cur] = t
        self.emit(chain, **u)
        if post_pool:
            # both bivariate stages of the 2x2 window in one pass (kernels_simt.cu bipool2_kernel)
            a, b = post_pool
            pn = g.nodes[a]
            tp = self.tensor(sh[b])
            self.fused.update(post_pool)
            self.value[b] = tp
            self.emit([a, b], kind=L.UNIT_LOCALPOOL, in_=t, out=tp, npad=cpad_for(sh[b][0]), kh=2, kw=2,
                      stride=2, pad=0, pool=L.POOL_BI2, pool_deg=pn.degree,
                      pool_order=0 if pn.axis == "w" else 1, pool_off=self.cast_pair(a, b))

    def lower_linear(self, nid: str):
        g = self.g
        node = g.nodes[nid]
        pred = self.preds[nid][0]
        pn = g.nodes[pred]
        if pred in self.value:
            src, mode = self.value[pred], 0
        elif pred in self.fused and isinstance(pn, FlattenNode):
            src, mode = self.value[self.preds[pred][0]], 1
        elif pred in self.fused and isinstance(pn, AvgPoolNode):
            src, mode = self.value[self.preds[pred][0]], 2
        else:
            src, mode = self.value[pred], 0
        k, n = node.weight.shape
        u = dict(kind=L.UNIT_LINEAR, in_=src, cin=n, cout=k, in_mode=mode, npad=cpad_for(k))
        if mode == 2:
            u["in_div_off"] = self.cast(pred, "divisor")
        u["w_off"] = self.cast(nid, "weight")
        u["b_off"] = self.cast(nid, "bias")
        chain = [pred, nid] if mode else [nid]
        cur = nid
        nxt = self.single(cur)
        if nxt and isinstance(g.nodes[nxt[0]], PolyActNode):
            cur = nxt[0]
            chain.append(cur)
            self.fused.add(cur)
            u["poly_deg"] = g.nodes[cur].degree
            u["poly_off"] = self.cast(cur, "coeffs")
        t = self.tensor(self.shapes[cur])
        u["out"] = t
        self.value[cur] = t
        self.emit(chain, **u)

    def lower_eltwise(self, nid: str):
        g = self.g
        node = g.nodes[nid]
        preds = self.preds[nid]
        t = self.tensor(self.shapes[nid])
        u = dict(out=t, in_=self.value[preds[0]], npad=cpad_for(self.shapes[nid][0]))
        if isinstance(node, PolyActNode):
            u.update(kind=L.UNIT_POLY, poly_deg=node.degree, poly_off=self.cast(nid, "coeffs"))
        elif isinstance(node, AddNode):
            u.update(kind=L.UNIT_ADD, in2=self.value[preds[1]])
        elif isinstance(node, PolySkipNode):
            u.update(kind=L.UNIT_POLYSKIP, in2=self.value[preds[1]], res_off=self.cast(nid, "coeffs"))
        elif isinstance(node, BatchNormNode):
            u.update(kind=L.UNIT_AFFINE, affine_off=self.affine(nid))
        elif isinstance(node, LocalPoolNode):
            u.update(kind=L.UNIT_LOCALPOOL, kh=node.k, kw=node.k, stride=node.stride, pad=node.padding,
                     pool_off=self.cast(nid, "divisor"))
        elif isinstance(node, BiPoolNode):
            u.update(kind=L.UNIT_BIPOOL, pool_deg=node.degree, pool_order=0 if node.axis == "w" else 1,
                     pool_off=self.cast(nid, "coeffs"))
        else:
            raise GraphError(f"node {nid!r}: no GPU lowering for kind {node.kind!r}")
        self.value[nid] = t
        self.emit([nid], **u)


def _schedule(units: List[Dict], unit_nodes: List[List[str]]):
    """Topologically order units by the tensors they read and write."""
    writer = {u["out"]: i for i, u in enumerate(units) if u.get("out", -1) >= 0}
    deps = []
    for u in units:
        ins = [u.get("in_", -1), u.get("in2", -1)]
        deps.append({writer[t] for t in ins if t >= 0 and t in writer})
    done, order = set(), []
    while len(order) < len(units):
        progressed = False
        for i in range(len(units)):
            if i not in done and deps[i] <= done:
                done.add(i)
                order.append(i)
                progressed = True
        if not progressed:
            raise GraphError("fused units form a dependency cycle")
    return [units[i] for i in order], [unit_nodes[i] for i in order]


def lower(g: ModelGraph, use_tc: bool = True, _layout=None) -> Lowered:
    shapes = g.validate()
    slots, chunks, size, scalar = _layout or build_master(g, shapes)
    b = _Builder(g, slots, size, use_tc).run()
    units, unit_nodes = _schedule(b.units, b.unit_nodes)
    lw = Lowered(graph=g, shapes=shapes, tensors=b.tensors, units=units, unit_nodes=unit_nodes,
                 slots=slots, master_size=size, pack_ops=b.pack, packed_size=max(b.packed, ALIGN),
                 input_tensor=b.input_tensor, output_tensor=b.output_tensor,
                 out_shape=tuple(b.output_shape), scalar=scalar)
    lw._chunks = chunks
    return lw


# ---------------------------------------------------------------------------
# neutral model format straight into the master layout
# ---------------------------------------------------------------------------

def load_lowered(path: str, use_tc: bool = True) -> Tuple[Lowered, np.ndarray]:
    """levnet's neutral JSON model (reference graph.py:433-539, written by
    exporter neutral.py:57-91 / graph.save_model) -> (Lowered, float64
    master) without copying any parameter into per-node arrays.

    The base64 blob is decoded once.  The graph the lowering walks holds
    read-only views into the blob (graph.load_model_views), and the master
    is ONE vectorised gather: the master layout (build_master) is computed
    on blob indices instead of values -- element i of the blob enters as
    the code i + 2 (exact in float64), the layout's zero padding stays 0 and
    its BatchNorm std padding 1 -- then master = [0, 1, blob...][code].
    Byte-identical to master_array(lower(load_model(path))) -- see
    tests/test_loader.py."""
    g, blob, specs = load_model_views(path)
    shapes = g.validate()

    def get(node, field):
        off, shape = specs[node.id][field]
        n = int(np.prod(shape)) if shape else 1
        return np.arange(off + 2, off + 2 + n, dtype=np.float64).reshape(shape)

    slots, chunks, size, scalar = build_master(g, shapes, get)
    code = master_array(chunks, size).astype(np.int64)
    ext = np.empty(blob.size + 2)
    ext[0], ext[1] = 0.0, 1.0
    ext[2:] = blob
    master = ext[code]
    lw = lower(g, use_tc=use_tc, _layout=(slots, chunks, size, scalar))
    lw._chunks = None  # the chunks hold encoded indices; the master is the gathered array
    return lw, master
