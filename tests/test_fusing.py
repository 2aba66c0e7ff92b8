"""Node fusing (P2F, reference transforms.py:62-277), host half: the fused
graph's structure from fusing.fuse_structure must be node-for-node and
edge-for-edge what the reference wrote (golden fixture_P2F), with the
reference's rewrite list; the single-site host helpers (the reference API)
match the oracle's rules.  The parameter values come from the device
program (tests/test_gpu_parity.py)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import max_param_rel_diff
from oracle import levnet_oracle as O
from paper_2509_22857_b200 import configs, fusing
from paper_2509_22857_b200.graph import BatchNormNode, ConvNode, PolyActNode, load_model


def _case(name):
    m = json.loads((GOLDEN / "manifest.json").read_text())
    return next(c for c in m["cases"] if c["name"] == name)


def test_structure_matches_reference_p2f():
    case = _case("fixture_P2F")
    before = load_model(str(GOLDEN / case["before"]))
    want = load_model(str(GOLDEN / case["after"]))
    work, applied, plan = fusing.fuse_structure(before)
    assert [[r, list(ids)] for r, ids in applied] == case["rewrites"]
    assert list(work.nodes) == list(want.nodes)
    assert [type(n) for n in work.nodes.values()] == [type(n) for n in want.nodes.values()]
    assert work.edges == want.edges
    assert len(plan) == len(applied)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_structure_matches_oracle_shuffled(seed):
    """Site order shuffled (the reference's rng option) on a ResNet with
    BatchNorms: the same fused structure as the oracle's fuse_pass."""
    g = load_model(str(GOLDEN / _case("fixture_P2F")["before"]))
    a, applied_a, _ = fusing.fuse_structure(g, np.random.default_rng(seed))
    b, applied_b = O.fuse_pass(g, np.random.default_rng(seed))
    assert applied_a == [(r, tuple(i)) for r, i in applied_b]
    assert list(a.nodes) == list(b.nodes) and a.edges == b.edges


def test_host_helpers_match_oracle(rng):
    c = 8
    bn = BatchNormNode("bn", rng.uniform(0.5, 2, c), rng.normal(0, 1, c), rng.normal(0, 1, c), rng.uniform(0.5, 2, c))
    bn2 = BatchNormNode("bn2", rng.uniform(0.5, 2, c), rng.normal(0, 1, c), rng.normal(0, 1, c),
                        rng.uniform(0.5, 2, c))
    act = PolyActNode("act", [rng.normal(0, 1, c), np.float64(0.7), rng.uniform(0.1, 0.5, c)])
    conv = ConvNode("conv", rng.normal(0, 1, (c, 3, 3, 3)), rng.normal(0, 1, c), 1, 1)
    pairs = [(fusing.fuse_bn_act(bn, act), O.fuse_bn_act(bn, act)),
             (fusing.fuse_bn_conv(conv, bn), O.fuse_bn_conv(conv, bn)),
             (fusing.fuse_skip_bn_bn(bn, bn2, act), O.fuse_skip_bn_bn(bn, bn2, act)),
             (fusing.fuse_skip_identity(bn, act), O.fuse_skip_identity(bn, act))]
    from helpers import node_tensors
    for got, want in pairs:
        tg, tw = node_tensors(got), node_tensors(want)
        assert tg.keys() == tw.keys()
        for k in tg:
            np.testing.assert_allclose(np.broadcast_to(tg[k], np.shape(tw[k])), tw[k], rtol=1e-13, atol=1e-13)
    with pytest.raises(fusing.FusionError):
        fusing.fuse_bn_act(bn, PolyActNode("a3", [np.float64(0), np.float64(1), np.float64(0), np.float64(1)]))


def test_compose_affine_any_degree(rng):
    """P(s x + t) by the binomial expansion, checked pointwise (degree 1..6)."""
    for d in range(1, 7):
        c = rng.normal(0, 1, d + 1)
        s, t = rng.uniform(0.5, 2), rng.normal()
        x = rng.uniform(-2, 2, 25)
        got = np.polynomial.polynomial.polyval(x, fusing.compose_affine(c, s, t))
        np.testing.assert_allclose(got, np.polynomial.polynomial.polyval(s * x + t, c), rtol=1e-11, atol=1e-11)
