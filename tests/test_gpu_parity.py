"""GPU parity: the B200 path against the float64 oracle (pinned to the
reference by tests/golden) -- forward outputs and redistributed parameters.

Tolerances (north star): forward rel 1e-4 / abs 1e-5 in float32 compute and
reference-style max|a-b|/max|a| <= 1e-4; redistributed weights and
coefficients within 1e-6 relative of the reference (float64 on device, so
in practice ~1e-15).
"""

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import chain, max_param_rel_diff, rel_err
from oracle import levnet_oracle as O
from paper_2509_22857_b200 import transforms as T
from paper_2509_22857_b200.graph import (AvgPoolNode, BiPoolNode, ConvNode, FlattenNode, InputNode,
                                         LinearNode, LocalPoolNode, OutputNode, PolyActNode, load_model)
from paper_2509_22857_b200.runtime import Engine, reference_eval

pytestmark = pytest.mark.gpu

FWD_RTOL, FWD_ATOL = 1e-4, 1e-5


def _load(rel):
    return load_model(str(GOLDEN / rel))


def assert_forward_close(got, want, name=""):
    got = np.asarray(got, dtype=np.float64)
    assert np.all(np.isfinite(got)), name
    np.testing.assert_allclose(got, want, rtol=FWD_RTOL, atol=FWD_ATOL, err_msg=name)
    assert rel_err(got, want) <= FWD_RTOL, name


@pytest.mark.parametrize("impl", [0, 1])
def test_forward_matches_golden(cuda, golden, impl):
    import torch
    manifest, arrays = golden
    for case in manifest["cases"]:
        if case["kind"] != "eval":
            continue
        g = _load(case["model"])
        x = arrays[case["name"] + "/x"]
        eng = Engine(g, impl=impl)
        y = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
        assert_forward_close(y, arrays[case["name"] + "/y"], case["name"])


def test_reference_eval_dropin(cuda, golden):
    manifest, arrays = golden
    case = next(c for c in manifest["cases"] if c["name"] == "rn20_fixture")
    g = _load(case["model"])
    x = arrays["rn20_fixture/x"][0]
    assert_forward_close(reference_eval(g, x), arrays["rn20_fixture/y"][0])


def test_reference_eval_loop_reuses_engine(cuda, golden):
    """A levnet caller looping reference_eval per image (the reference's
    usage, transforms.py:768-769) pays the lowering / upload / plan capture
    once: on RN20, 100 calls cost far less than 100 engine builds, every
    result matches the oracle, and an edited graph is lowered again."""
    import time
    import torch
    from paper_2509_22857_b200 import configs
    from paper_2509_22857_b200 import runtime as R
    g = configs.build("resnet20")
    xs = configs.make_input(configs.CONFIGS["resnet20"], batch=8)
    want = O.eval_batch(g, xs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Engine(g).forward(torch.from_numpy(xs[:1].astype(np.float32)).cuda())
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    R.clear_engine_cache()
    assert_forward_close(reference_eval(g, xs[0]), want[0])
    hits0 = R._ENGINES.hits
    t0 = time.perf_counter()
    for i in range(100):
        y = reference_eval(g, xs[i % len(xs)])
    loop = time.perf_counter() - t0
    assert_forward_close(y, want[99 % len(xs)])
    assert R._ENGINES.hits - hits0 == 100
    assert loop < 0.3 * 100 * build, (loop, build)  # each cached call < 30 % of a fresh build
    # editing a parameter array invalidates the cached engine
    conv = next(n for n in g.nodes.values() if isinstance(n, ConvNode))
    conv.bias = conv.bias + 1.0
    misses = R._ENGINES.misses
    reference_eval(g, xs[0])
    assert R._ENGINES.misses == misses + 1


def test_forward_host_rejects_bad_buffers(cuda, golden):
    """forward_host / forward_host_many check shapes, dtypes and staging
    sizes before libpcnn copies batch * C * H * W floats."""
    import torch
    from paper_2509_22857_b200.graph import GraphError
    manifest, arrays = golden
    g = _load(next(c for c in manifest["cases"] if c["name"] == "rn20_fixture")["model"])
    x = arrays["rn20_fixture/x"].astype(np.float32)
    eng = Engine(g)
    with pytest.raises(GraphError):
        eng.forward_host(x[:, :, :-1])  # wrong spatial shape
    with pytest.raises(GraphError):
        eng.forward_host(x, x_dev=torch.empty(1, device="cuda"))  # staging too small
    with pytest.raises(GraphError):
        eng.forward_host_many([torch.from_numpy(x.astype(np.float64))])  # float64 batch
    with pytest.raises(GraphError):
        eng.forward_host_many([torch.from_numpy(x)[:, :, ::2]])  # strided / wrong shape


def test_forward_host_e2e_matches_device(cuda, golden):
    import torch
    manifest, arrays = golden
    g = _load(next(c for c in manifest["cases"] if c["name"] == "rn20_fixture")["model"])
    x = arrays["rn20_fixture/x"].astype(np.float32)
    eng = Engine(g)
    a = eng.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    b = eng.forward_host(x)
    # a global pool fused into a conv epilogue sums with float atomics: runs
    # agree to rounding, not bit for bit
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-7)


def test_graph_replay_equals_eager(cuda, golden):
    import torch
    manifest, arrays = golden
    g = _load(next(c for c in manifest["cases"] if c["name"] == "rn18_poly2_s1")["model"])
    x = torch.from_numpy(arrays["rn18_poly2_s1/x"].astype(np.float32)).cuda()
    eng = Engine(g)
    a = eng.forward(x, use_graph=False).cpu().numpy()
    b = eng.forward(x, use_graph=True).cpu().numpy()
    c = eng.forward(x, use_graph=True).cpu().numpy()
    # (fused global pools sum with float atomics: equal to rounding)
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(b, c, rtol=1e-6, atol=1e-7)


def _ext_graph(rng, kind):
    if kind == "lenet_like":
        return chain([InputNode("in", 1, 12, 12),
                      ConvNode("c1", rng.normal(0, 0.3, (6, 1, 3, 3)), rng.normal(0, 0.1, 6), 1, 0),
                      PolyActNode("a1", [np.float64(0.1), np.float64(0.5), np.float64(0.3)]),
                      LocalPoolNode("p1", 2, 2, 0, np.float64(0.25)),
                      FlattenNode("f"),
                      LinearNode("fc1", rng.normal(0, 0.2, (7, 150)), rng.normal(0, 0.1, 7)),
                      PolyActNode("a2", [rng.normal(0, 0.3, 7), rng.normal(0, 0.3, 7), rng.uniform(0.1, 0.5, 7)]),
                      LinearNode("fc2", rng.normal(0, 0.3, (3, 7)), rng.normal(0, 0.1, 3)),
                      OutputNode("out")])
    if kind == "bipool":
        d = 4
        c1 = rng.normal(0, 0.2, (d + 1, d + 1, 8))
        c2 = rng.normal(0, 0.2, (d + 1, d + 1))
        i, j = np.indices((d + 1, d + 1))
        c1[(i + j) > d] = 0
        c2[(i + j) > d] = 0
        c1[d, 0] = rng.uniform(0.05, 0.3, 8)
        c2[d, 0] = 0.2
        return chain([InputNode("in", 3, 8, 8),
                      ConvNode("c1", rng.normal(0, 0.3, (8, 3, 3, 3)), rng.normal(0, 0.1, 8), 1, 1),
                      PolyActNode("a1", [np.float64(0.0), np.float64(0.6), np.float64(0.2), np.float64(0.1)]),
                      BiPoolNode("pw", "w", c1), BiPoolNode("ph", "h", c2),
                      ConvNode("c2", rng.normal(0, 0.3, (16, 8, 3, 3)), rng.normal(0, 0.1, 16), 1, 1),
                      AvgPoolNode("gp", 16, np.float64(1 / 16)),
                      LinearNode("fc", rng.normal(0, 0.3, (5, 16)), rng.normal(0, 0.1, 5)),
                      OutputNode("out")])
    if kind == "stem_pool":
        return chain([InputNode("in", 3, 15, 15),
                      ConvNode("c1", rng.normal(0, 0.2, (32, 3, 7, 7)), rng.normal(0, 0.1, 32), 2, 3),
                      PolyActNode("a1", [rng.normal(0, 0.3), rng.normal(0, 0.3), rng.normal(0, 0.3),
                                         rng.normal(0, 0.3), np.float64(0.1)]),
                      LocalPoolNode("p", 3, 2, 1, np.float64(1 / 9)),
                      ConvNode("c2", rng.normal(0, 0.1, (64, 32, 3, 3)), rng.normal(0, 0.1, 64), 1, 1),
                      AvgPoolNode("gp", 16, np.float64(1 / 16)),
                      LinearNode("fc", rng.normal(0, 0.3, (10, 64)), rng.normal(0, 0.1, 10)),
                      OutputNode("out")])
    raise KeyError(kind)


@pytest.mark.parametrize("kind", ["lenet_like", "bipool", "stem_pool"])
@pytest.mark.parametrize("impl", [0, 1])
def test_extension_nodes_forward(cuda, kind, impl):
    import torch
    rng = np.random.default_rng(3)
    g = _ext_graph(rng, kind)
    shape = g.validate()["in"]
    x = rng.normal(0, 1, (9,) + shape)
    want = O.eval_batch(g, x)
    got = Engine(g, impl=impl).forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert_forward_close(got, want, kind)


# -- redistribution parity ----------------------------------------------------

def _replay_gpu(case, before):
    name = case["name"]
    if name == "fwd_act_conv":
        return T.redistribute_forward(before, "act")
    if name == "fwd_act_conv_u2.5":
        return T.redistribute_forward(before, "act", 2.5)
    if name in ("bwd_conv_act", "bwd_conv_act_deg3"):
        return T.redistribute_backward(before, "act")
    if name == "fwd_pool_linear":
        return T.redistribute_forward(before, "pool")
    if name == "rn20_forward_sweep":
        return T.redistribute_sweep(before, "forward")[0]
    if name.startswith("rn20_forward_"):
        return T.redistribute_forward(before, name[len("rn20_forward_"):])
    if name.startswith("rn20_backward_"):
        return T.redistribute_backward(before, name[len("rn20_backward_"):])
    if name.startswith("fixture_"):
        return T.apply_pipeline(before, name.split("_", 1)[1])[0]
    if name.endswith("_P2FR"):
        return T.apply_pipeline(before, "P2FR")[0]
    if name == "rn20_poly4_pass":
        return T.redistribute_pass(before)[0]
    raise KeyError(name)


def test_redistribution_matches_reference(cuda, golden):
    manifest, arrays = golden
    n = 0
    for case in manifest["cases"]:
        if case["kind"] != "rewrite":
            continue
        before, want = _load(case["before"]), _load(case["after"])
        got = _replay_gpu(case, before)
        assert max_param_rel_diff(got, want) <= 1e-6, case["name"]
        n += 1
    assert n >= 15


def test_pipeline_rewrite_lists(cuda, golden):
    manifest, _ = golden
    for case in manifest["cases"]:
        if "rewrites" in case and case["name"].startswith("fixture_"):
            _, rep = T.apply_pipeline(_load(case["before"]), case["name"].split("_", 1)[1])
            assert [[a, list(b)] for a, b in rep.rewrites] == case["rewrites"], case["name"]
            assert [rep.depth_before, rep.depth_after] == case["depth"]


def test_refusals_match_reference(cuda, golden):
    manifest, _ = golden
    for err in manifest["errors"]:
        g = _load(err["model"])
        fn = T.redistribute_forward if err["direction"] == "forward" else T.redistribute_backward
        with pytest.raises(T.TransformError) as ei:
            fn(g, err["donor"])
        assert str(ei.value) == err["message"]


def test_sweep_acceptance_sets(cuda, golden):
    manifest, _ = golden
    case = next(c for c in manifest["cases"] if c["name"] == "rn20_forward_sweep")
    g = _load(case["before"])
    for direction in ("forward", "backward"):
        _, applied, _ = T.redistribute_sweep(g, direction)
        assert applied == [n for n in g.topo_order() if n in manifest["rn20_donors"][direction]]


def test_redistributed_model_is_equivalent_on_gpu(cuda, golden):
    manifest, _ = golden
    case = next(c for c in manifest["cases"] if c["name"] == "fixture_P2FR")
    before = _load(case["before"])
    after, _ = T.apply_pipeline(before, "P2FR")
    rep = T.check_equivalence(before, after, n_inputs=64, rtol=1e-4, seed=3)
    assert rep.passed and rep.argmax_match_rate == 1.0


def test_extension_redistribution_matches_oracle(cuda):
    rng = np.random.default_rng(5)
    for kind in ("lenet_like", "bipool", "stem_pool"):
        g = _ext_graph(rng, kind)
        for direction in ("forward", "backward"):
            want, applied_o, _ = O.redistribute_sweep(g, direction, allow_negative_leading=True)
            got, applied, _ = T.redistribute_sweep(g, direction, allow_negative_leading=True)
            assert applied == applied_o, (kind, direction)
            assert max_param_rel_diff(got, want) <= 1e-12, (kind, direction)


def test_engine_from_model_file(cuda, golden, tmp_path):
    """Engine.from_model_file (blob gathered straight into the master,
    lowering.load_lowered) runs the same network as Engine(load_model())."""
    import torch
    manifest, arrays = golden
    case = next(c for c in manifest["cases"] if c["name"] == "rn20_fixture")
    path = str(GOLDEN / case["model"])
    x = torch.from_numpy(arrays["rn20_fixture/x"].astype(np.float32)).cuda()
    a = Engine(load_model(path)).forward(x).cpu().numpy()
    e = Engine.from_model_file(path)
    b = e.forward(x).cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-7)
    assert_forward_close(b, arrays["rn20_fixture/y"], "from_model_file")
    assert max_param_rel_diff(e.to_graph(), load_model(path)) == 0.0


def test_forward_host_space_to_depth_input(cuda):
    """A 7x7/s2 stem ingested as 2x2 space-to-depth blocks: the host-buffer
    entry points copy the user's NCHW image (batch * C * H * W floats), not
    the ingest tensor's (4C, H/2+1, W/2+1) size."""
    import torch
    from paper_2509_22857_b200 import configs
    g = configs.build("resnet18", hw=64, calib_batch=4)
    x = configs.make_input(configs.CONFIGS["resnet18"], batch=8, hw=64).astype(np.float32)
    eng = Engine(g)
    assert eng.lw.tensors[eng.lw.input_tensor].c == 12  # the space-to-depth ingest tensor
    want = eng.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_allclose(eng.forward_host(x), want, rtol=1e-6, atol=1e-7)
    outs = eng.forward_host_many([x, x[::-1].copy()])
    np.testing.assert_allclose(outs[0].numpy(), want, rtol=1e-6, atol=1e-7)
    assert rel_err(O.eval_batch(g, x[:2]), want[:2].astype(np.float64)) <= 1e-4


@pytest.mark.parametrize("model", ["models/rn20_fixture.json", "models/rn18_poly2_s1.json",
                                   "models/ckpt_rn20_w4_ref.json"])
def test_device_fusing_matches_reference(cuda, model):
    """P2F node fusing with every parameter computed by one device launch
    (fusing.py) = the reference's host algebra (oracle fuse_pass, pinned to
    the reference): same structure, parameters within 1e-12 relative."""
    from paper_2509_22857_b200 import fusing
    g = _load(model)
    got, applied = fusing.fuse_pass(g)
    want, applied_ref = O.fuse_pass(g)
    assert applied and [(r, tuple(i)) for r, i in applied_ref] == applied
    assert got.edges == want.edges
    assert max_param_rel_diff(got, want) <= 1e-12
    x = np.random.default_rng(4).uniform(-1, 1, (4,) + g.validate()[g.input_id()])
    assert rel_err(O.eval_batch(got, x), O.eval_batch(g, x)) <= 1e-10
