"""Node fusing (the P2F step of apply_pipeline) with the parameter algebra on
the GPU.

Reference: levnet transforms.py:62-277 -- BatchNorm folded into the
preceding conv (:76-86) or into the following degree-2 activation (:62-73),
and a residual join of BatchNorm'd branches followed by a degree-2
activation rewritten as one bivariate quadratic PolySkip node (:89-101), the
three rule families applied to disjoint sites until none is left
(:104-277).

The split between host and device follows the redistribution pass:

* host -- the graph STRUCTURE: which sites fuse (same priorities and claims
  as the reference, so the fused graph is node-for-node and edge-for-edge
  the reference's) and the surgery on nodes and edges.  No parameter value
  is computed here: fused nodes get placeholder arrays of the right shape.
* device -- every parameter of the fused graph, in ONE pcnn_redistribute
  launch over a buffer holding [fused master | original master]:
  per-channel BatchNorm slopes and offsets s = gamma / std, t = beta - s mean
  (phase a), conv weights scaled per output row by s while being copied
  (phase b factor chains), conv biases s b + t, activation coefficients of
  P(s x + t) and the six PolySkip coefficients (phase a vector algebra),
  every untouched parameter copied into its slot of the fused layout.

``fuse_pass`` returns the fused graph (downloaded from the device master)
and the applied sites in the reference's (rule, ids) form; ``apply_pipeline``
(P2F, P2FR) runs on it.  The single-site helpers (fuse_bn_act, fuse_bn_conv,
fuse_skip_bn_bn, fuse_skip_identity) keep the reference's host API.
"""

from __future__ import annotations

from math import comb
from typing import Dict, List, Optional, Tuple

import numpy as np

from .graph import (AddNode, BatchNormNode, ConvNode, ModelGraph, PolyActNode, PolySkipNode, PS_KEYS,
                    copy_node)


class FusionError(Exception):
    pass


# ---------------------------------------------------------------------------
# host algebra (reference API; the device program below computes the same)
# ---------------------------------------------------------------------------

def compose_affine(coeffs, s, t) -> List[np.ndarray]:
    """Coefficients of P(s x + t) for P = sum_k c_k x^k (binomial expansion:
    c'_j = s^j sum_{k >= j} C(k, j) t^(k-j) c_k)."""
    c = [np.asarray(x, dtype=np.float64) for x in coeffs]
    s, t = np.asarray(s, dtype=np.float64), np.asarray(t, dtype=np.float64)
    d = len(c) - 1
    return [s ** j * sum(comb(k, j) * t ** (k - j) * c[k] for k in range(j, d + 1)) for j in range(d + 1)]


def _need_quadratic(act: PolyActNode, what: str) -> None:
    if act.degree != 2:
        raise FusionError(f"{what} needs a degree-2 activation, got degree {act.degree}")


def fuse_bn_act(bn: BatchNormNode, act: PolyActNode) -> PolyActNode:
    """Activation after BatchNorm: P(b1 x + b0) (reference transforms.py:62-73)."""
    _need_quadratic(act, "batchnorm folding into an activation")
    return PolyActNode(act.id, compose_affine(act.coeffs, bn.b1, bn.b0))


def fuse_bn_conv(conv: ConvNode, bn: BatchNormNode) -> ConvNode:
    """BatchNorm after a conv: rows scaled by b1, bias b1 b + b0 (transforms.py:76-86)."""
    if bn.gamma.shape[0] != conv.weight.shape[0]:
        raise FusionError(f"batchnorm width {bn.gamma.shape[0]} does not match "
                          f"{conv.weight.shape[0]} conv output channels")
    return ConvNode(conv.id, conv.weight * bn.b1[:, None, None, None], bn.b1 * conv.bias + bn.b0,
                    conv.stride, conv.padding)


def join_quadratic(coeffs, sx, tx, sy, ty) -> Dict[str, np.ndarray]:
    """P(sx x + tx + sy y + ty) for a quadratic P as the six PolySkip
    monomials (transforms.py:89-101): with u = sx x + sy y, k = tx + ty,
    P = c2 u^2 + (2 c2 k + c1) u + P(k)."""
    c0, c1, c2 = (np.asarray(x, dtype=np.float64) for x in coeffs)
    sx, sy = np.asarray(sx, dtype=np.float64), np.asarray(sy, dtype=np.float64)
    k = np.asarray(tx, dtype=np.float64) + np.asarray(ty, dtype=np.float64)
    lin = 2.0 * c2 * k + c1
    shape = np.broadcast_shapes(np.shape(sx), np.shape(sy), np.shape(c2))
    full = lambda v: np.broadcast_to(v, shape).astype(np.float64)
    return {"x2": full(c2 * sx * sx), "y2": full(c2 * sy * sy), "xy": full(2.0 * c2 * sx * sy),
            "x": full(sx * lin), "y": full(sy * lin), "c": full((c2 * k + c1) * k + c0)}


def fuse_skip_bn_bn(bnX: BatchNormNode, bnY: BatchNormNode, act: PolyActNode) -> PolySkipNode:
    _need_quadratic(act, "skip fusion")
    return PolySkipNode(act.id, join_quadratic(act.coeffs, bnX.b1, bnX.b0, bnY.b1, bnY.b0))


def fuse_skip_identity(bnX: BatchNormNode, act: PolyActNode) -> PolySkipNode:
    _need_quadratic(act, "skip fusion")
    return PolySkipNode(act.id, join_quadratic(act.coeffs, bnX.b1, bnX.b0, 1.0, 0.0))


# ---------------------------------------------------------------------------
# structure: sites and surgery (host)
# ---------------------------------------------------------------------------

def _sole_consumer(g: ModelGraph, nid: str) -> Optional[str]:
    cons = g.consumers_of(nid)
    return cons[0] if len(cons) == 1 else None


def _is_quadratic(g: ModelGraph, nid: Optional[str]) -> bool:
    return nid is not None and isinstance(g.nodes[nid], PolyActNode) and g.nodes[nid].degree == 2


def find_sites(g: ModelGraph) -> List[Tuple[str, Tuple[str, ...]]]:
    """The reference's rule priorities over disjoint sites: residual joins
    first (a BatchNorm whose only consumer is the join is claimed by it),
    then conv + BatchNorm, then BatchNorm + activation on what is left."""
    order = g.topo_order()
    joins, convs, acts = [], [], []
    claimed, folded = set(), set()
    for nid in order:
        node = g.nodes[nid]
        if isinstance(node, AddNode):
            act = _sole_consumer(g, nid)
            if not _is_quadratic(g, act):
                continue
            x, y = g.inputs_of(nid)
            own = [isinstance(g.nodes[q], BatchNormNode) and [c for c, _ in g.consumer_edges(q)] == [nid]
                   for q in (x, y)]
            if own[0] and own[1]:
                joins.append(("fuse_skip_bn_bn", (x, y, nid, act)))
                claimed |= {x, y}
            elif own[0]:
                joins.append(("fuse_skip_identity", (x, nid, act)))
                claimed.add(x)
            elif own[1]:
                joins.append(("fuse_skip_identity_y", (y, nid, act)))
                claimed.add(y)
    for nid in order:
        if isinstance(g.nodes[nid], ConvNode):
            bn = _sole_consumer(g, nid)
            if bn is not None and isinstance(g.nodes[bn], BatchNormNode) and bn not in claimed:
                convs.append(("fuse_bn_conv", (nid, bn)))
                folded.add(bn)
    for nid in order:
        if isinstance(g.nodes[nid], BatchNormNode) and nid not in claimed and nid not in folded:
            act = _sole_consumer(g, nid)
            if _is_quadratic(g, act):
                acts.append(("fuse_bn_act", (nid, act)))
    return joins + convs + acts


def _drop_first(edges: List[Tuple[str, str]], gone: List[Tuple[str, str]]) -> List[Tuple[str, str]]:
    """Remove one occurrence of each pair in `gone`, keeping the order."""
    pending = list(gone)
    out = []
    for e in edges:
        if e in pending:
            pending.remove(e)
        else:
            out.append(e)
    return out


def _only_input(g: ModelGraph, nid: str) -> str:
    return g.inputs_of(nid)[0]


def apply_structure(g: ModelGraph, rule: str, ids: Tuple[str, ...]) -> Dict:
    """Rewire g for one site (the reference's surgery: removed nodes' edges
    dropped in place, new input edges of the surviving node appended) and
    return what the device program needs: the operands of the rule."""
    if rule == "fuse_bn_conv":
        conv, bn = ids
        g.edges = [(conv if s == bn else s, d) for s, d in _drop_first(g.edges, [(conv, bn)])]
        del g.nodes[bn]
        return {"conv": conv, "bn": bn}
    if rule == "fuse_bn_act":
        bn, act = ids
        src = _only_input(g, bn)
        g.edges = _drop_first(g.edges, [(src, bn), (bn, act)])
        del g.nodes[bn]
        g.connect(src, act)
        g.nodes[act] = PolyActNode(act, [np.zeros(_width(g, act)) for _ in range(3)])
        return {"bn": bn, "act": act}
    if rule not in ("fuse_skip_bn_bn", "fuse_skip_identity", "fuse_skip_identity_y"):
        raise FusionError(f"unknown fusion rule {rule!r}")
    if rule == "fuse_skip_bn_bn":
        bx, by, add, act = ids
        gone = [bx, by]
        xs, ys = _only_input(g, bx), _only_input(g, by)
    elif rule == "fuse_skip_identity":
        bx, add, act = ids
        by = None
        gone = [bx]
        xs, ys = _only_input(g, bx), next(q for q in g.inputs_of(add) if q != bx)
    else:
        by, add, act = ids
        bx = None
        gone = [by]
        xs, ys = next(q for q in g.inputs_of(add) if q != by), _only_input(g, by)
    drop = [(add, act)]
    for b in gone:
        drop += [(_only_input(g, b), b), (b, add)]
    drop += [(q, add) for q in g.inputs_of(add) if q not in gone]
    width = _width(g, act)
    g.edges = _drop_first(g.edges, drop)
    for b in gone:
        del g.nodes[b]
    del g.nodes[add]
    g.connect(xs, act)
    g.connect(ys, act)
    g.nodes[act] = PolySkipNode(act, {k: np.zeros(width) for k in PS_KEYS})
    return {"bx": bx, "by": by, "act": act}


def _width(g: ModelGraph, nid: str) -> int:
    return g._infer_shapes()[nid][0]


# ---------------------------------------------------------------------------
# device program
# ---------------------------------------------------------------------------

class _Values:
    """Symbolic parameter values of the graph being fused: arena vectors
    (cpad long) for everything a rule touched, the original master slot for
    everything else; conv weights as (source offset, per-row factors)."""

    def __init__(self, prog, old_lw, base: int):
        self.p, self.old, self.base = prog, old_lw, base
        self.vecs: Dict[Tuple[str, str], object] = {}
        self.rows: Dict[str, List[object]] = {}  # conv id -> per-row weight factors

    def _slot(self, nid, name):
        return self.old.slots[nid][name]

    def cpad(self, nid: str) -> int:
        sl = self.old.slots[nid]
        if "bn" in sl:
            return sl["bn"].meta["cpad"]
        if "coeffs" in sl:
            return sl["coeffs"].meta["cpad"]
        return sl["bias"].n

    def get(self, nid: str, key: str, cp: int):
        if (nid, key) in self.vecs:
            return self.vecs[(nid, key)]
        p = self.p
        if key in ("gamma", "beta", "mean", "std"):
            s = self._slot(nid, "bn")
            return p.load(self.base + s.offset + ("gamma", "beta", "mean", "std").index(key) * cp, cp)
        if key == "bias":
            return p.load(self.base + self._slot(nid, "bias").offset, cp)
        s = self._slot(nid, "coeffs")
        i = int(key[1:]) if key[0] == "c" and key[1:].isdigit() else PS_KEYS.index(key)
        return p.load(self.base + s.offset + i * cp, cp)

    def slope_offset(self, bn: str, cp: int):
        """BatchNorm b1 = gamma / std, b0 = beta - b1 mean (graph.py BatchNormNode)."""
        p = self.p
        s = p.div(self.get(bn, "gamma", cp), self.get(bn, "std", cp))
        return s, p.sub(self.get(bn, "beta", cp), p.mul(s, self.get(bn, "mean", cp)))


def _emit_rule(vals: _Values, g_before: ModelGraph, rule: str, ops: Dict) -> None:
    p = vals.p
    if rule == "fuse_bn_conv":
        conv, bn = ops["conv"], ops["bn"]
        cp = vals.cpad(conv)
        s, t = vals.slope_offset(bn, cp)
        vals.rows.setdefault(conv, []).append(s)
        vals.vecs[(conv, "bias")] = p.add(p.mul(s, vals.get(conv, "bias", cp)), t)
        return
    if rule == "fuse_bn_act":
        bn, act = ops["bn"], ops["act"]
        cp = vals.cpad(bn)
        s, t = vals.slope_offset(bn, cp)
        c0, c1, c2 = (vals.get(act, f"c{k}", cp) for k in range(3))
        # c0' = (c2 t + c1) t + c0, c1' = s (2 c2 t + c1), c2' = s^2 c2
        ct = p.mul(c2, t)
        vals.vecs[(act, "c0")] = p.add(p.mul(p.add(ct, c1), t), c0)
        vals.vecs[(act, "c1")] = p.mul(s, p.add(p.add(ct, ct), c1))
        vals.vecs[(act, "c2")] = p.mul(p.mul(s, s), c2)
        return
    act = ops["act"]
    cp = None
    for b in (ops["bx"], ops["by"]):
        if b is not None:
            cp = vals.cpad(b)
    one, zero = p.fill(1.0, cp), p.fill(0.0, cp)
    sx, tx = vals.slope_offset(ops["bx"], cp) if ops["bx"] is not None else (one, zero)
    sy, ty = vals.slope_offset(ops["by"], cp) if ops["by"] is not None else (one, zero)
    c0, c1, c2 = (vals.get(act, f"c{k}", cp) for k in range(3))
    k = p.add(tx, ty)
    lin = p.add(p.mul(p.add(c2, c2), k), c1)
    c2sx, c2sy = p.mul(c2, sx), p.mul(c2, sy)
    out = {"x2": p.mul(c2sx, sx), "y2": p.mul(c2sy, sy), "xy": p.add(p.mul(c2sx, sy), p.mul(c2sx, sy)),
           "x": p.mul(sx, lin), "y": p.mul(sy, lin), "c": p.add(p.mul(p.add(p.mul(c2, k), c1), k), c0)}
    for key in ("c0", "c1", "c2"):
        vals.vecs.pop((act, key), None)
    for key, v in out.items():
        vals.vecs[(act, key)] = v


def fuse_structure(g: ModelGraph, rng: Optional[np.random.Generator] = None):
    """Host half of fuse_pass: the fused graph's nodes and edges (fused
    nodes with placeholder parameters), the applied sites, and each site's
    operands for the device program."""
    g.validate()
    work = ModelGraph()
    for node in g.nodes.values():
        work.add(copy_node(node))
    work.edges = list(g.edges)
    applied: List[Tuple[str, Tuple[str, ...]]] = []
    plan: List[Tuple[str, Dict]] = []
    while True:
        sites = find_sites(work)
        if not sites:
            break
        if rng is not None:
            rng.shuffle(sites)
        for rule, ids in sites:
            plan.append((rule, apply_structure(work, rule, ids)))
            applied.append((rule, ids))
    work.validate()
    return work, applied, plan


def fuse_pass(g: ModelGraph, rng: Optional[np.random.Generator] = None, engine=None):
    """Fuse until no site is left (reference fuse_pass, transforms.py:250-277):
    structure on the host, every parameter on the device (one launch).
    Returns (fused graph, [(rule, ids), ...]); engine: an Engine of g to reuse."""
    import torch
    from . import _lib as L
    from .lowering import lower
    from .runtime import Engine
    from .transforms import Program, run_program_on

    work, applied, plan = fuse_structure(g, rng)
    if not applied:
        return g.copy(), applied
    old = engine or Engine(g)
    new_lw = lower(work)
    n_new = new_lw.master_size
    prog = Program(new_lw)
    vals = _Values(prog, old.lw, n_new)
    for rule, ops in plan:
        _emit_rule(vals, g, rule, ops)
    # every slot of the fused layout: computed vectors, scaled conv rows, or copies
    for nid, slots in new_lw.slots.items():
        node = work.nodes[nid]
        for name, s in slots.items():
            src = old.lw.slots.get(nid, {}).get(name)
            if isinstance(node, ConvNode) and name == "weight" and nid in vals.rows:
                m = s.meta
                row = (m["kp"], m["npad"], 1, 1, 1)
                for f in vals.rows[nid]:
                    prog.factor(s.offset, s.n, f, False, row)
                prog.src_of[s.offset] = n_new + src.offset
            elif isinstance(node, ConvNode) and name == "bias" and (nid, "bias") in vals.vecs:
                prog.set_from(s.offset, s.n, vals.vecs[(nid, "bias")])
            elif isinstance(node, PolyActNode) and (nid, "c0") in vals.vecs:
                cp = s.meta["cpad"]
                for k in range(3):
                    prog.set_from(s.offset + k * cp, cp, vals.vecs[(nid, f"c{k}")])
            elif isinstance(node, PolySkipNode) and (nid, "x2") in vals.vecs:
                cp = s.meta["cpad"]
                for i, key in enumerate(PS_KEYS):
                    prog.set_from(s.offset + i * cp, cp, vals.vecs[(nid, key)])
            else:
                if src is None or src.n != s.n:
                    raise FusionError(f"node {nid!r}: no source for parameter slot {name!r}")
                prog.copy(s.offset, s.n, n_new + src.offset)
    both = torch.empty(n_new + old.lw.master_size, dtype=torch.float64, device=old.device)
    both[n_new:] = old.master
    run_program_on(both, prog, old.device)
    new = Engine(work, lowered=new_lw, master=np.zeros(n_new))
    new.master.copy_(both[:n_new])
    new.repack()
    out = new.to_graph()
    out.validate()
    return out, applied
