"""Test helpers: graph parameter comparison and small graph builders."""

import numpy as np

from paper_2509_22857_b200.graph import (
    BatchNormNode, BiPoolNode, ConvNode, InputNode, LinearNode, ModelGraph,
    OutputNode, PolyActNode, PolySkipNode, AvgPoolNode, LocalPoolNode)


def node_tensors(node):
    """Flat dict name -> float64 array of every parameter of a node."""
    if isinstance(node, (ConvNode, LinearNode)):
        return {"weight": node.weight, "bias": node.bias}
    if isinstance(node, BatchNormNode):
        return {"gamma": node.gamma, "beta": node.beta, "mean": node.mean, "std": node.std}
    if isinstance(node, PolyActNode):
        return {f"c{i}": np.asarray(c) for i, c in enumerate(node.coeffs)}
    if isinstance(node, PolySkipNode):
        return {k: np.asarray(v) for k, v in node.coeffs.items()}
    if isinstance(node, (AvgPoolNode, LocalPoolNode)):
        return {"divisor": np.asarray(node.divisor)}
    if isinstance(node, BiPoolNode):
        return {"coeffs": np.asarray(node.coeffs)}
    return {}


def max_param_rel_diff(a: ModelGraph, b: ModelGraph, check_shapes=True):
    """Largest relative difference over every parameter of two same-shaped
    graphs (relative to the max magnitude of each tensor)."""
    assert set(a.nodes) == set(b.nodes)
    assert a.edges == b.edges
    worst = 0.0
    for nid in a.nodes:
        ta, tb = node_tensors(a.nodes[nid]), node_tensors(b.nodes[nid])
        assert ta.keys() == tb.keys(), nid
        for k in ta:
            x, y = np.asarray(ta[k], dtype=np.float64), np.asarray(tb[k], dtype=np.float64)
            if check_shapes:
                assert x.shape == y.shape, (nid, k, x.shape, y.shape)
            x, y = np.broadcast_arrays(x, y)
            scale = max(float(np.max(np.abs(x))) if x.size else 0.0, 1e-300)
            worst = max(worst, float(np.max(np.abs(x - y))) / scale if x.size else 0.0)
    return worst


def rel_err(got, want):
    return float(np.max(np.abs(got - want)) / max(float(np.max(np.abs(want))), 1e-12))


def chain(nodes):
    g = ModelGraph()
    for n in nodes:
        g.add(n)
    for a, b in zip(nodes, nodes[1:]):
        g.connect(a.id, b.id)
    g.validate()
    return g
