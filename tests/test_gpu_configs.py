"""The five benchmark configurations end to end on the GPU: the config's
redistribution sweeps run on the device (one cooperative launch each) and
match the float64 oracle's per-donor sweep parameter for parameter; the
redistributed model's batched forward (auto precision = tcgen05 fp16x2 where
supported) matches the oracle at rel 1e-4 / abs 1e-5; and, because several
configs' logits are dominated by a constant offset, the
batch-centred logits -- the input-dependent signal -- must match too."""

import numpy as np
import pytest

from helpers import max_param_rel_diff, rel_err
from oracle import levnet_oracle as O
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import transforms as T
from paper_2509_22857_b200.runtime import Engine

pytestmark = pytest.mark.gpu

def _device_sweeps(g, cfg):
    eng = Engine(g)
    cur = g
    for direction in cfg.redistribution:
        accepted, _ = T.plan_sweep(eng, cur, direction, allow_negative_leading=cfg.allow_negative_leading)
        prog = T.compile_sweep(eng, cur, direction, accepted, cfg.allow_negative_leading)
        T.run_program(eng, prog)
        cur = eng.to_graph()
    return eng, cur


def _oracle_sweeps(g, cfg):
    for direction in cfg.redistribution:
        g, _, _ = O.redistribute_sweep(g, direction, allow_negative_leading=cfg.allow_negative_leading)
    return g


@pytest.mark.parametrize("name", list(configs.CONFIGS))
def test_config_redistributed_forward(cuda, name):
    """Every image of the measured batch (64 / 256 / 512 / 128 / 64) against
    the float64 oracle: rel 1e-4 / abs 1e-5 elementwise, the reference's
    max|a-b|/max|a| <= 1e-4 (transforms.py:768-772), and the batch-centred
    logits within 1e-3 of their range -- the oracle runs over the host cores
    (oracle/pool.py), so there is no reason to sample."""
    import torch
    from oracle.pool import OraclePool
    cfg = configs.CONFIGS[name]
    g = configs.build(name)
    eng, got_g = _device_sweeps(g, cfg)
    want_g = _oracle_sweeps(g, cfg)
    assert max_param_rel_diff(got_g, want_g) <= 1e-6, name

    x = configs.make_input(cfg)
    assert len(x) == cfg.batch
    y = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert np.all(np.isfinite(y)), name
    with OraclePool(want_g) as pool:
        want = pool.eval(x)
    np.testing.assert_allclose(y, want, rtol=1e-4, atol=1e-5, err_msg=name)
    assert rel_err(y, want) <= 1e-4, name
    # input-dependent part of the logits (RN18 / VGG logits are ~99.7 % constant)
    cg, cw = y - y.mean(0), want - want.mean(0)
    assert np.abs(cw).max() > 0, name
    assert np.abs(cg - cw).max() <= 1e-3 * np.abs(cw).max(), (name, np.abs(cg - cw).max() / np.abs(cw).max())
    # per image: the argmax agrees wherever the oracle's top-2 margin exceeds the tolerance
    top2 = np.sort(want, axis=1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 1e-4 * np.abs(want).max()
    assert np.all(np.argmax(y, 1)[clear] == np.argmax(want, 1)[clear]), name
    # the redistributed model is the original function (float64 oracle, full batch)
    with OraclePool(g) as pool:
        orig = pool.eval(x)
    assert rel_err(want, orig) <= 1e-8, name


@pytest.mark.parametrize("name", ["resnet20", "resnet18", "resnet20_deg8"])
def test_flag_synchronised_launches_match(cuda, name):
    """options.flag_sync = 1 (per-tile completion counters instead of whole-grid
    griddepcontrol ordering, api.cu build_flags) computes the same logits:
    every tile does the same arithmetic, only the global-pool atomics may
    add in another order."""
    import ctypes
    import torch
    from paper_2509_22857_b200 import _lib as L
    cfg = configs.CONFIGS[name]
    g, _, _ = T.redistribute_sweep(configs.build(name), cfg.redistribution[0],
                                   allow_negative_leading=cfg.allow_negative_leading)
    x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
    base = Engine(g).forward(x).double().cpu().numpy()
    eng = Engine(g, options=L.PlanOptions.default(flag_sync=1))
    fn = L.lib().pcnn_plan_flags
    fn.argtypes = [ctypes.c_void_p]
    assert fn(eng.plan(cfg.batch).handle) == 1, name
    for _ in range(3):  # graph replays reuse the zeroed counters
        got = eng.forward(x).double().cpu().numpy()
        # (flag mode keeps whole tiles; the default plan may split tiles
        # stream-K, which sums the same products in another order)
        assert rel_err(got, base) <= 1e-5, name


def test_forward_host_many_pipeline(cuda):
    """pcnn_forward_host_many (H2D of batch i+1 overlapping batch i's
    forward, two staging buffers) returns, for every batch, the logits the
    plain device forward computes for it."""
    import torch
    cfg = configs.CONFIGS["resnet20"]
    g, _, _ = T.redistribute_sweep(configs.build("resnet20"), "forward")
    eng = Engine(g)
    xs = [configs.make_input(cfg, batch=64, seed=s).astype(np.float32) for s in (2, 5, 7, 9, 11)]
    outs = eng.forward_host_many(xs)
    for x, o in zip(xs, outs):
        want = eng.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_err(o.numpy(), want) <= 1e-6
    # odd counts and a single batch take the same path
    one = eng.forward_host_many(xs[:1])
    assert rel_err(one[0].numpy(), outs[0].numpy()) <= 1e-6


def test_check_equivalence_replicas_single_rank(cuda):
    """Without a process group check_equivalence_replicas is
    check_equivalence (same inputs, same report)."""
    g = configs.build("lenet5")
    rg, _, _ = T.redistribute_sweep(g, "forward")
    a = T.check_equivalence(g, rg, n_inputs=32, rtol=1e-4)
    b = T.check_equivalence_replicas(g, rg, n_inputs=32, rtol=1e-4)
    assert a.passed and b.passed
    # default rtol: the float32-reachable DEVICE_RTOL, never a silent failure
    c = T.check_equivalence(g, rg, n_inputs=32)
    assert c.passed and c.max_rel_err == a.max_rel_err
    with pytest.warns(RuntimeWarning):
        T.check_equivalence(g, rg, n_inputs=8, rtol=1e-8)
    assert abs(a.max_rel_err - b.max_rel_err) <= 1e-7 and a.argmax_match_rate == b.argmax_match_rate


@pytest.mark.parametrize("name", ["resnet20", "resnet18", "vgg11"])
def test_streamk_matches_whole_tiles(cuda, name):
    """Stream-K forced onto every layer with <= 2 rounds of tiles
    (options.streamk_fill = 2: RN20 stage 3, RN18 stages 3-4, VGG's 8x8..2x2
    layers, fused projections included) computes what whole tiles compute,
    up to the summation order of the split chunks."""
    import torch
    cfg = configs.CONFIGS[name]
    g = configs.build(name)
    for d in cfg.redistribution:
        g, _, _ = T.redistribute_sweep(g, d, allow_negative_leading=cfg.allow_negative_leading)
    x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
    from paper_2509_22857_b200 import _lib as L
    base = Engine(g, options=L.PlanOptions.default(streamk=0)).forward(x).double().cpu().numpy()
    eng = Engine(g, options=L.PlanOptions.default(streamk_fill=2.0))
    for _ in range(2):
        got = eng.forward(x).double().cpu().numpy()
        assert rel_err(got, base) <= 1e-5, name


@pytest.mark.parametrize("name", ["lenet5", "resnet20"])
def test_compare_report(cuda, name, tmp_path):
    """The GPU compare report (reference cli.py:554-629's transform-equivalence
    check over 1000 inputs through forward_host_many, plus the per-unit
    precision table): passes on the configs' redistributions, agrees with
    check_equivalence on the common inputs, and the CLI writes the JSON and
    exits 0."""
    import json
    from paper_2509_22857_b200 import compare
    cfg = configs.CONFIGS[name]
    g = configs.build(name)
    rg = g
    for d in cfg.redistribution:
        rg, _, _ = T.redistribute_sweep(rg, d, allow_negative_leading=cfg.allow_negative_leading)
    rep = compare.compare_report(g, rg, n_inputs=1000)
    eq, prec = rep["checks"]
    assert rep["passed"] and eq["passed"] and eq["n_inputs"] == 1000
    assert eq["max_rel_err"] <= 1e-4 and eq["argmax_match_rate"] >= 0.99
    small = T.check_equivalence(g, rg, n_inputs=100)
    assert small.max_rel_err <= eq["max_rel_err"] + 1e-7  # the first 100 inputs are the same draws
    # a whole-network launch (LeNet: impl 7, fp32 CUDA cores) stores only the logits
    assert len(prec["units"]) >= (1 if prec["units"][0]["impl"] == 7 else 3)
    assert prec["logits_max_rel_err_vs_fp32"] <= 1e-4
    out = tmp_path / "r.json"
    assert compare.main(["--config", name, "--n-inputs", "300", "--json", str(out)]) == 0
    assert json.loads(out.read_text())["passed"]


@pytest.mark.parametrize("images", [1, 2])
@pytest.mark.parametrize("name", ["resnet20", "resnet20_deg8"])
def test_image_resident_runs_match(cuda, name, images):
    """options.image_blocks: runs of stride-1 3x3 convs computed in one launch
    with whole images' activations in shared memory (conv_ss.cu
    conv_blk_kernel) give the logits of the per-layer launches (the same
    per-element arithmetic; only the global-pool atomics may add in another
    order) with fewer launches; images = 2 keeps two images per CTA resident
    and alternates between them layer by layer."""
    import torch
    from paper_2509_22857_b200 import _lib as L
    cfg = configs.CONFIGS[name]
    g = configs.build(name)
    for d in cfg.redistribution:
        g, _, _ = T.redistribute_sweep(g, d, allow_negative_leading=cfg.allow_negative_leading)
    x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
    base = Engine(g, options=L.PlanOptions.default(image_blocks=0))
    eng = Engine(g, options=L.PlanOptions.default(image_blocks=images))
    want = base.forward(x).double().cpu().numpy()
    for _ in range(2):
        got = eng.forward(x).double().cpu().numpy()
        assert rel_err(got, want) <= 1e-5, name
    assert eng.plan(cfg.batch).launches() < base.plan(cfg.batch).launches()
    assert eng.fallbacks == 0


@pytest.mark.parametrize("batch", [1, 64, 300])
def test_whole_network_launch_matches(cuda, batch):
    """options.fused_net: LeNet's ingest, convs with their fused poly + 2x2
    pools, dense layers and logits in ONE launch (net_fused.cu, whole images
    and every parameter in shared memory) agree with the oracle and with the
    unit-by-unit launches; batch 300 > the grid makes CTAs loop over images."""
    import torch
    from paper_2509_22857_b200 import _lib as L
    cfg = configs.CONFIGS["lenet5"]
    g = configs.build("lenet5")
    for d in cfg.redistribution:
        g, _, _ = T.redistribute_sweep(g, d)
    x = configs.make_input(cfg, batch=batch)
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    fused = Engine(g)
    layered = Engine(g, options=L.PlanOptions.default(fused_net=0))
    got = fused.forward(xt).double().cpu().numpy()
    assert fused.plan(batch).launches() == 1 and fused.plan(batch).unit_impl(1) == 7
    assert layered.plan(batch).unit_impl(1) != 7
    want = O.eval_batch(g, x)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)
    assert rel_err(got, layered.forward(xt).double().cpu().numpy()) <= 1e-5
    # graph replay and the host-buffer entry point run the same launch
    assert rel_err(fused.forward(xt, use_graph=True).double().cpu().numpy(), got) <= 1e-7
    outs = fused.forward_host_many([torch.from_numpy(x.astype(np.float32))])
    assert rel_err(outs[0].double().numpy(), got) <= 1e-7


@pytest.mark.gpu
@pytest.mark.parametrize("opts", [{"epi_pairs": 1}, {"epi_pairs": 3}, {"epi_pairs": 4}, {"ss_pair": 0},
                                  {"ss_wide": 0}, {"ss_wide": 2}, {"scratch_cb4": 1}],
                         ids=lambda o: ",".join(f"{k}={v}" for k, v in o.items()))
@pytest.mark.parametrize("name", ["resnet18", "vgg11"])
def test_halo_tile_option_variants_match(cuda, name, opts):
    """Every halo-tile scheduling option ships tested: epilogue warpgroup
    pairs on no / 64-channel / every tile (options.epi_pairs 1 / 3 / 4),
    CTA-pair tiles off (options.ss_pair) and the producer's single- or
    multi-lane bulk-copy issue (options.ss_wide) and the 4-channel-block
    scratch map between a conv and its local pool (options.scratch_cb4)
    change who drains or stages a tile or where a scratch value lives, never
    the arithmetic: logits equal the default plan's (the
    global-pool atomics may add in another order)."""
    import torch
    from paper_2509_22857_b200 import _lib as L
    cfg = configs.CONFIGS[name]
    g = configs.build(name)
    for d in cfg.redistribution:
        g, _, _ = T.redistribute_sweep(g, d, allow_negative_leading=cfg.allow_negative_leading)
    x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
    base = Engine(g)
    want = base.forward(x).double().cpu().numpy()
    eng = Engine(g, options=L.PlanOptions.default(**opts))
    for _ in range(2):
        got = eng.forward(x).double().cpu().numpy()
        assert rel_err(got, want) <= 1e-5, (name, opts)
    # the fp16-range rescue (one float32 rerun + rescale on VGG's first batch) is the plan's, not the option's
    assert eng.fallbacks == base.fallbacks
