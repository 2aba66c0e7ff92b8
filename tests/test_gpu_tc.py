"""tcgen05 conv kernels against the float64 oracle on single fused conv
units of every supported shape class, and against the SIMT kernel: impl=2
forces 3xTF32 (kind::tf32, A from TMEM), impl=3 fp16x2 (kind::f16, three fp16
products on power-of-two scaled weights), impl=5 fp16x2 with both operands in
shared memory (halo tiles of split activations; stride-1 3x3/1x1 only, other
shapes fall back to impl 3); plan creation fails loudly if no tcgen05 kernel
supports the shape."""

import numpy as np
import pytest

from helpers import chain, rel_err
from oracle import levnet_oracle as O
from paper_2509_22857_b200.graph import (AddNode, AvgPoolNode, BiPoolNode, ConvNode, InputNode, LinearNode,
                                         LocalPoolNode, ModelGraph, OutputNode, PolyActNode)
from paper_2509_22857_b200.runtime import Engine

pytestmark = pytest.mark.gpu

IMPLS = pytest.mark.parametrize("impl", [2, 3, 5], ids=["tf32x3", "f16x2", "f16x2_smem"])


def _check_impls(impls, impl, ss_ok=True):
    """impl 3/5 requests land on the shared-memory kernel (5) when the shape
    and input format allow, else on the TMEM-A kernel (3)."""
    if impl == 2:
        assert impls == {2}
    elif impl == 5 and ss_ok:
        assert impls == {5}
    else:
        assert impls <= {3, 5}

SHAPES = [
    # cin, cout, k, stride, pad, hw, batch
    (3, 16, 3, 1, 1, 32, 4),
    (16, 16, 3, 1, 1, 16, 8),
    (16, 32, 3, 2, 1, 16, 8),
    (32, 64, 3, 1, 1, 8, 16),
    (64, 128, 3, 1, 1, 8, 4),
    (128, 256, 3, 2, 1, 8, 4),
    (256, 512, 3, 1, 1, 4, 4),
    (16, 32, 1, 2, 0, 16, 8),
    (3, 64, 7, 2, 3, 30, 2),
    (6, 16, 5, 1, 0, 12, 8),
]


def conv_graph(rng, cin, cout, k, s, p, hw, tail=(), gain=1.0):
    """Conv (+ fused tail); gain sets the conv output std (the configs keep
    polynomial inputs near 0.3 by calibration, see configs.py)."""
    nodes = [InputNode("in", cin, hw, hw),
             ConvNode("conv", rng.normal(0, gain / np.sqrt(cin * k * k), (cout, cin, k, k)),
                      rng.normal(0, 0.1, cout), s, p)]
    nodes += list(tail)
    nodes.append(OutputNode("out"))
    return chain(nodes)


def run(g, x, impl, **options):
    import torch
    from paper_2509_22857_b200 import _lib as L
    eng = Engine(g, impl=impl, options=L.PlanOptions.default(**options) if options else None)
    y = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda())
    # 6: halo-tile arithmetic inside an image-resident run -- the same kernel math as 5
    impls = {5 if m == 6 else m for m in (eng.plan(x.shape[0]).unit_impl(i) for i, u in enumerate(eng.lw.units)
                                         if u["kind"] == 2)}
    return y.double().cpu().numpy(), impls


@IMPLS
@pytest.mark.parametrize("shape", SHAPES, ids=[f"{s[0]}x{s[1]}k{s[2]}s{s[3]}h{s[5]}" for s in SHAPES])
def test_tc_plain_conv(cuda, shape, impl):
    cin, cout, k, s, p, hw, batch = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    g = conv_graph(rng, cin, cout, k, s, p, hw)
    x = rng.normal(0, 1, (batch, cin, hw, hw))
    want = O.eval_batch(g, x)
    got, impls = run(g, x, impl)
    _check_impls(impls, impl, s in (1, 2) and (cin % 16 == 0 or cin <= 8) and k in (1, 3) and p == k // 2)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)
    simt, _ = run(g, x, 1)
    # fp32-class accuracy from the 3-product split: within a small factor of plain fp32 FMA
    assert rel_err(got, want) <= max(4 * rel_err(simt, want), 2e-6)


def _poly(rng, c, d):
    cs = [rng.normal(0, 0.3, c) for _ in range(d)] + [rng.uniform(0.05, 0.3, c)]
    return PolyActNode("act", cs)


@IMPLS
@pytest.mark.parametrize("deg", [2, 4, 8])
def test_tc_conv_poly(cuda, deg, impl):
    rng = np.random.default_rng(deg)
    g = conv_graph(rng, 16, 32, 3, 1, 1, 16, [_poly(rng, 32, deg)], gain=0.5)
    x = rng.normal(0, 1, (8, 16, 16, 16))
    want = O.eval_batch(g, x)
    got, impls = run(g, x, impl)
    _check_impls(impls, impl)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)


@IMPLS
def test_tc_conv_pools(cuda, impl):
    rng = np.random.default_rng(11)
    d = 4
    c = rng.normal(0, 0.2, (d + 1, d + 1, 64))
    i, j = np.indices((d + 1, d + 1))
    c[(i + j) > d] = 0
    for tail in ([_poly(rng, 64, 2), LocalPoolNode("pool", 2, 2, 0, np.float64(0.25))],
                 [_poly(rng, 64, 3), BiPoolNode("pw", "w", c), BiPoolNode("ph", "h", c.copy())],
                 [_poly(rng, 64, 3), BiPoolNode("ph", "h", c), BiPoolNode("pw", "w", c.copy())],
                 [_poly(rng, 64, 2), AvgPoolNode("gp", 64, np.float64(1 / 64))]):
        g = conv_graph(rng, 32, 64, 3, 1, 1, 8, tail, gain=0.3)
        x = rng.normal(0, 1, (16, 32, 8, 8))
        want = O.eval_batch(g, x)
        got, impls = run(g, x, impl)
        _check_impls(impls, impl, tail[-1].kind in ("avgpool",))
        np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)


@IMPLS
def test_tc_conv_residual(cuda, impl):
    rng = np.random.default_rng(12)
    g = ModelGraph()
    g.add(InputNode("in", 32, 8, 8))
    g.add(ConvNode("ca", rng.normal(0, 0.1, (32, 32, 3, 3)), rng.normal(0, 0.1, 32), 1, 1))
    g.add(PolyActNode("aa", [np.float64(0.0), np.float64(0.5), np.float64(0.2)]))
    g.add(ConvNode("cb", rng.normal(0, 0.1, (32, 32, 3, 3)), rng.normal(0, 0.1, 32), 1, 1))
    g.add(AddNode("j"))
    g.add(PolyActNode("aj", [rng.normal(0, 0.1, 32), rng.normal(0.5, 0.1, 32), rng.uniform(0.05, 0.3, 32)]))
    g.add(OutputNode("out"))
    for s_, d_ in (("in", "ca"), ("ca", "aa"), ("aa", "cb"), ("cb", "j"), ("in", "j"), ("j", "aj"), ("aj", "out")):
        g.connect(s_, d_)
    g.validate()
    x = rng.normal(0, 1, (16, 32, 8, 8))
    want = O.eval_batch(g, x)
    got, impls = run(g, x, impl)
    _check_impls(impls, impl)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)


def test_tc_matches_simt_on_resnet20(cuda):
    import torch
    from paper_2509_22857_b200 import configs
    g = configs.build("resnet20")
    x = configs.make_input(configs.CONFIGS["resnet20"], batch=32)
    tc, impls = run(g, x, 0)
    assert 5 in impls and impls <= {3, 5}  # auto picks fp16x2, shared-memory kernel where possible
    simt, _ = run(g, x, 1)
    want = O.eval_batch(g, x[:4])
    np.testing.assert_allclose(tc[:4], want, rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(tc, simt, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("shape", [(16, 32, 3, 1, 1, 16, 8), (64, 128, 3, 1, 1, 8, 4)], ids=["n32", "n128"])
def test_f16x2_overflow_rows_recomputed(cuda, shape):
    """float32 input tensors (options.split = 0) into the TMEM-A fp16x2 kernel:
    inputs beyond the fp16 range (|x| >= 65520) poison their pixel's
    accumulator row; the epilogue redoes exactly those rows in fp32."""
    cin, cout, k, s, p, hw, batch = shape
    rng = np.random.default_rng(5)
    g = conv_graph(rng, cin, cout, k, s, p, hw)
    x = rng.normal(0, 1, (batch, cin, hw, hw))
    x[0, 0, 3, 4] = 1.0e6
    x[1, cin - 1, 0, 0] = -7.0e4
    x[batch - 1, :, hw - 1, :] = 3.0e5
    want = O.eval_batch(g, x)
    got, impls = run(g, x, 3, split=0)
    assert impls == {3}
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5 * np.abs(want).max())


@pytest.mark.parametrize("wscale", [1e-6, 1e4])
def test_f16x2_weight_scaling(cuda, wscale):
    """Weights far outside fp16's comfortable range are packed with a power of
    two scale and unscaled in the epilogue."""
    rng = np.random.default_rng(6)
    g = conv_graph(rng, 32, 64, 3, 1, 1, 8, gain=wscale)
    x = rng.normal(0, 1, (8, 32, 8, 8))
    want = O.eval_batch(g, x)
    got, impls = run(g, x, 3)
    assert impls <= {3, 5}
    simt, _ = run(g, x, 1)
    assert rel_err(got, want) <= max(4 * rel_err(simt, want), 2e-6)


def test_split_tensors_and_overflow_fallback(cuda):
    """fp16x2 convs chained through split-format (hi/lo fp16) activations; an
    activation outside the fp16 range sets the plan status, the engine
    recomputes the batch on float32 tensors and rescales the offending
    tensors so later batches stay on the fast path."""
    import torch
    rng = np.random.default_rng(21)
    g = ModelGraph()
    g.add(InputNode("in", 16, 8, 8))
    g.add(ConvNode("ca", rng.normal(0, 0.1, (32, 16, 3, 3)), rng.normal(0, 0.1, 32), 1, 1))
    g.add(PolyActNode("aa", [np.float64(0.0), np.float64(0.5), np.float64(0.2)]))
    g.add(ConvNode("cb", rng.normal(0, 0.1, (32, 32, 3, 3)), rng.normal(0, 0.1, 32), 1, 1))
    g.add(ConvNode("cd", rng.normal(0, 0.1, (32, 16, 1, 1)), rng.normal(0, 0.1, 32), 1, 0))
    g.add(AddNode("j"))
    g.add(PolyActNode("aj", [rng.normal(0, 0.1, 32), rng.normal(0.5, 0.1, 32), rng.uniform(0.05, 0.3, 32)]))
    g.add(AvgPoolNode("gp", 64, np.float64(1 / 64)))
    g.add(LinearNode("fc", rng.normal(0, 0.2, (10, 32)), rng.normal(0, 0.1, 10)))
    g.add(OutputNode("out"))
    for s_, d_ in (("in", "ca"), ("ca", "aa"), ("aa", "cb"), ("cb", "j"), ("in", "cd"), ("cd", "j"),
                   ("j", "aj"), ("aj", "gp"), ("gp", "fc"), ("fc", "out")):
        g.connect(s_, d_)
    g.validate()
    eng = Engine(g)
    x = rng.normal(0, 1, (16, 16, 8, 8))
    plan = eng.plan(16)
    assert any(plan.tensor_split(t) for t in range(len(eng.lw.tensors)))
    got = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert eng.fallbacks == 0
    np.testing.assert_allclose(got, O.eval_batch(g, x), rtol=1e-4, atol=1e-5)
    # an input value beyond fp16 range: the ingest flags it, the rerun is exact
    x[3, 2, 4, 4] = 1.0e5
    want = O.eval_batch(g, x)
    got = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert eng.fallbacks == 1
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5 * np.abs(want).max())
    # the rerun recalibrated: the input tensor is now stored scaled by 2^-k
    assert eng.scale_log2.min() < 0
    got_h = eng.forward_host(x.astype(np.float32)).astype(np.float64)
    assert eng.fallbacks == 1  # the fast path handles it now
    np.testing.assert_allclose(got_h, want, rtol=1e-4, atol=1e-5 * np.abs(want).max())
    got = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert eng.fallbacks == 1
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5 * np.abs(want).max())


BAND_CASES = [
    # cin, cout, k(conv), hw, batch, pool: ("local", k, s, p) | ("bi", degree, axis-first)
    (16, 64, 3, 20, 6, ("local", 3, 2, 1)),
    (16, 64, 3, 17, 5, ("local", 3, 2, 1)),   # odd conv rows / columns
    (32, 128, 3, 12, 7, ("local", 2, 2, 0)),
    (3, 64, 7, 40, 3, ("local", 3, 2, 1)),    # space-to-depth 7x7/s2 stem + 3x3/s2 pool (ResNet-18's)
    (16, 64, 3, 16, 9, ("bi", 4, "w")),
    (64, 128, 3, 10, 6, ("bi", 3, "h")),
    (32, 256, 3, 8, 6, ("bi", 2, "w")),       # two n-tiles
]


@pytest.mark.parametrize("case", BAND_CASES, ids=[f"{c[0]}x{c[1]}k{c[2]}h{c[3]}{c[5][0]}" for c in BAND_CASES])
def test_band_pooled_epilogue(cuda, case):
    """A conv (+ polynomial) followed by a local k x k / s pool or a 2x2
    bivariate pool runs as ONE halo-tile launch (conv_ss.cu band mode: the
    unpooled map never leaves the SM) and matches the oracle; the float32
    fallback plans (TMEM-A 3xTF32 / SIMT with a scratch map and a pooling
    launch) compute the same."""
    from paper_2509_22857_b200 import _lib as L
    cin, cout, k, hw, batch, pool = case
    rng = np.random.default_rng(31)
    stride, pad = (2, 3) if k == 7 else (1, k // 2)
    poly = PolyActNode("act", [rng.normal(0, 0.3, cout), rng.normal(0.6, 0.1, cout), rng.uniform(0.05, 0.3, cout)])
    if pool[0] == "local":
        _, pk, ps, pp = pool
        tail = [poly, LocalPoolNode("pool", pk, ps, pp, np.float64(1.0 / (pk * pk)))]
    else:
        _, d, first = pool
        second = "h" if first == "w" else "w"

        def coeffs():
            c = rng.normal(0, 0.2, (d + 1, d + 1, cout))
            i, j = np.indices((d + 1, d + 1))
            c[(i + j) > d] = 0.0
            c[d, 0] = rng.uniform(0.05, 0.3, cout)
            return c
        tail = [poly, BiPoolNode("p1", first, coeffs()), BiPoolNode("p2", second, coeffs())]
    g = conv_graph(rng, cin, cout, k, stride, pad, hw, tail=tail, gain=0.5)
    x = rng.normal(0, 1, (batch, cin, hw, hw))
    want = O.eval_batch(g, x)
    import torch
    eng = Engine(g, options=L.PlanOptions.default(band_pool=1))
    got = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    plan = eng.plan(batch)
    conv_units = [i for i, u in enumerate(eng.lw.units) if u["kind"] == L.UNIT_CONV]
    assert len(conv_units) == 1 and eng.lw.units[conv_units[0]]["pool"] in (L.POOL_LOCAL, L.POOL_BI2)
    assert plan.unit_impl(conv_units[0]) == 5
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5 * max(1.0, np.abs(want).max()))
    # default plan: the conv into scratch, then a pooling launch
    e0 = Engine(g)
    y0 = e0.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert e0.plan(batch).unit_impl(conv_units[0]) == 5 and e0.plan(batch).launches() == plan.launches() + 1
    np.testing.assert_allclose(y0, want, rtol=1e-4, atol=1e-5 * max(1.0, np.abs(want).max()))
    for impl in (1, 4):
        e2 = Engine(g, impl=impl)
        y2 = e2.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
        assert e2.plan(batch).unit_impl(conv_units[0]) in (1, 2)
        np.testing.assert_allclose(y2, want, rtol=1e-4, atol=1e-5 * max(1.0, np.abs(want).max()))
