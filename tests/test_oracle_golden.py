"""Pin the CPU oracle to the real reference (CPU only).

Every case in ``tests/golden/manifest.json`` was produced by running the
reference ``levnet`` package (see ``tests/golden/make_golden.py``).  The
oracle must reproduce those outputs; the forward and the rewrites restate the
same float64 operations in the same order, so they are compared at 1e-13.
"""

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import chain, max_param_rel_diff, rel_err
from oracle import levnet_oracle as O
from paper_2509_22857_b200.graph import (
    BiPoolNode, FlattenNode, InputNode, LinearNode, LocalPoolNode, OutputNode,
    PS_KEYS, load_model)


def _load(rel):
    return load_model(str(GOLDEN / rel))


def _cases(manifest, kind):
    return [c for c in manifest["cases"] if c["kind"] == kind]


def test_manifest_has_cases(golden):
    manifest, arrays = golden
    assert len(_cases(manifest, "eval")) >= 15
    assert len(_cases(manifest, "rewrite")) >= 15


def test_forward_matches_reference(golden):
    manifest, arrays = golden
    for case in _cases(manifest, "eval"):
        g = _load(case["model"])
        xs, ys = arrays[case["name"] + "/x"], arrays[case["name"] + "/y"]
        got = O.eval_batch(g, xs)
        np.testing.assert_allclose(got, ys, rtol=1e-13, atol=1e-300, err_msg=case["name"])


def _replay(case, before):
    """Re-run the reference function a rewrite case came from, on the oracle."""
    name = case["name"]
    if name == "fwd_act_conv":
        return O.redistribute_forward(before, "act")
    if name == "fwd_act_conv_u2.5":
        return O.redistribute_forward(before, "act", 2.5)
    if name in ("bwd_conv_act", "bwd_conv_act_deg3"):
        return O.redistribute_backward(before, "act")
    if name == "fwd_pool_linear":
        return O.redistribute_forward(before, "pool")
    if name.startswith("rn20_forward_sweep"):
        return None
    if name.startswith("rn20_forward_"):
        return O.redistribute_forward(before, name[len("rn20_forward_"):])
    if name.startswith("rn20_backward_"):
        return O.redistribute_backward(before, name[len("rn20_backward_"):])
    if name.startswith("fixture_"):
        return O.apply_pipeline(before, name.split("_", 1)[1])[0]
    if name.endswith("_P2FR"):
        return O.apply_pipeline(before, "P2FR")[0]
    if name == "rn20_poly4_pass":
        return O.redistribute_pass(before)[0]
    raise KeyError(name)


def test_rewrites_match_reference(golden):
    manifest, arrays = golden
    n = 0
    for case in _cases(manifest, "rewrite"):
        before, want = _load(case["before"]), _load(case["after"])
        got = _replay(case, before)
        if got is None:
            continue
        assert max_param_rel_diff(got, want) <= 1e-13, case["name"]
        n += 1
        if case["name"] + "/x" in arrays:
            ys = O.eval_batch(got, arrays[case["name"] + "/x"])
            np.testing.assert_allclose(ys, arrays[case["name"] + "/y_after"], rtol=1e-13)
    assert n >= 15


def test_forward_sweep_composition(golden):
    manifest, arrays = golden
    case = next(c for c in manifest["cases"] if c["name"] == "rn20_forward_sweep")
    before, want = _load(case["before"]), _load(case["after"])
    got, applied, refused = O.redistribute_sweep(before, "forward")
    assert applied == [n for n in before.topo_order() if n in manifest["rn20_donors"]["forward"]]
    assert max_param_rel_diff(got, want) <= 1e-13
    refused_ids = {r for r, _ in refused}
    assert refused_ids == {k.split(":", 1)[1] for k in manifest["rn20_donors"]["refused"]
                           if k.startswith("forward:")}


def test_backward_acceptance_set(golden):
    manifest, _ = golden
    case = next(c for c in manifest["cases"] if c["name"] == "rn20_forward_sweep")
    g = _load(case["before"])
    _, applied, _ = O.redistribute_sweep(g, "backward")
    assert applied == [n for n in g.topo_order() if n in manifest["rn20_donors"]["backward"]]


def test_pipeline_rewrites_lists(golden):
    manifest, _ = golden
    for case in _cases(manifest, "rewrite"):
        if "rewrites" not in case or not case["name"].startswith("fixture_"):
            continue
        before = _load(case["before"])
        _, rw = O.apply_pipeline(before, case["name"].split("_", 1)[1])
        assert [[a, list(b)] for a, b in rw] == case["rewrites"]


def test_error_messages_match_reference(golden):
    manifest, _ = golden
    for err in manifest["errors"]:
        g = _load(err["model"])
        fn = O.redistribute_forward if err["direction"] == "forward" else O.redistribute_backward
        with pytest.raises(O.TransformError) as ei:
            fn(g, err["donor"])
        assert str(ei.value) == err["message"]


def test_check_equivalence_matches_reference(golden):
    manifest, _ = golden
    e = manifest["equivalence"]
    rep = O.check_equivalence(_load(e["model_ref"]), _load(e["model_cand"]),
                              n_inputs=e["n_inputs"], rtol=1e-8, seed=e["seed"])
    assert rep.max_rel_err == pytest.approx(e["max_rel_err"], rel=1e-12, abs=1e-18)
    assert rep.argmax_match_rate == e["argmax_match_rate"]
    assert rep.passed == e["passed"]


# -- extension nodes against reference-expressible equivalents ---------------

@pytest.mark.parametrize("k,s,p", [(2, 2, 0), (3, 2, 1)])
def test_localpool_equals_diagonal_conv(golden, k, s, p):
    _, arrays = golden
    name = f"localpool_k{k}s{s}p{p}_as_conv"
    g = chain([InputNode("in", 3, 8, 8), LocalPoolNode("pool", k, s, p, np.float64(1.0 / (k * k))),
               OutputNode("out")])
    got = O.eval_batch(g, arrays[name + "/x"])
    assert rel_err(got, arrays[name + "/y"]) <= 1e-14


def test_flatten_linear_equals_full_conv(golden):
    _, arrays = golden
    name = "flatten_linear_as_conv"
    g = chain([InputNode("in", 4, 3, 3), FlattenNode("flat"),
               LinearNode("fc", arrays[name + "/w"], arrays[name + "/b"]), OutputNode("out")])
    got = O.eval_batch(g, arrays[name + "/x"])
    assert rel_err(got, arrays[name + "/y"]) <= 1e-13


def _ps_to_bivariate(ps):
    c = np.zeros((3, 3, len(ps["x"])))
    c[2, 0], c[0, 2], c[1, 1] = ps["x2"], ps["y2"], ps["xy"]
    c[1, 0], c[0, 1], c[0, 0] = ps["x"], ps["y"], ps["c"]
    return c


def test_bipool_degree2_equals_polyskip_tree(golden):
    _, arrays = golden
    name = "bipool2_as_polyskip"
    sw = {k: arrays[f"{name}/sw/{k}"] for k in PS_KEYS}
    sh = {k: arrays[f"{name}/sh/{k}"] for k in PS_KEYS}
    g = chain([InputNode("in", 3, 6, 6), BiPoolNode("pw", "w", _ps_to_bivariate(sw)),
               BiPoolNode("ph", "h", _ps_to_bivariate(sh)), OutputNode("out")])
    got = O.eval_batch(g, arrays[name + "/x"])
    assert rel_err(got, arrays[name + "/y"]) <= 1e-13


def test_bivariate_matches_polyval2d(rng):
    for d in (2, 3, 4):
        c = rng.standard_normal((d + 1, d + 1))
        i, j = np.indices(c.shape)
        c[(i + j) > d] = 0.0
        x, y = rng.uniform(-2, 2, 50), rng.uniform(-2, 2, 50)
        want = np.polynomial.polynomial.polyval2d(x, y, c)
        np.testing.assert_allclose(O.eval_bivariate(c, x, y), want, rtol=1e-12, atol=1e-12)


def test_batched_oracle_matches_per_image(golden):
    """eval_batch_fast (every node kernel with a batch axis; full-batch
    checker of the GPU tests and the bench parity field) = the per-image
    reference_eval restatement, on the reference-written golden forwards."""
    manifest, arrays = golden
    n = 0
    for case in manifest["cases"]:
        if case.get("kind") != "eval" or case["name"] + "/x" not in arrays:
            continue
        g = _load(case["model"])
        x = arrays[case["name"] + "/x"]
        want = arrays[case["name"] + "/y"]
        got = O.eval_batch_fast(g, x).reshape(want.shape)
        assert rel_err(got, O.eval_batch(g, x).reshape(want.shape)) <= 1e-13, case["name"]
        assert rel_err(got, want) <= 1e-13, case["name"]
        n += 1
    assert n >= 10
