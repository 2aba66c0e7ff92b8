"""Benchmark: images/s of the redistributed poly-CNN forward on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config resnet20] [--impl ours|reference]

One step = one fused forward of the redistributed network over one batch of
the configuration (input already resident in HBM), replayed as a CUDA graph
by libpcnn.  L2 is flushed (256 MiB write) between timed steps; each step is
bracketed by CUDA events on the launching stream and the per-step times are
summed; under torchrun the max over ranks is reported ("replicas only": each
rank runs its own batch, no collective on the data path).

The JSON line also carries
* e2e      -- the same metric through the C ABI with pinned host buffers
              (pcnn_forward_host_many: every step's input H2D and logits
              D2H inside the timed region, copies overlapping forwards);
* roofline -- the dominant kernel family against the fp32-accurate tensor
              rate of that kernel (fp16x2: bf16/3) or HBM bandwidth
              (MEASURED_PEAKS.json); its time per step is the union of its
              launches' intervals on the device timeline of every timed
              graph replay (pcnn_plan_timeline), so it cannot exceed the step;
* parity   -- the timed batch's logits against the float64 oracle, every
              image (oracle/pool.py over the host cores; the checker);
* secondary -- the same record for ResNet-18 (the second >= 60 % target
              config), measured in the same run;
* cpu_baseline -- the float64 oracle (restatement of levnet's
              reference_eval) on the host cores, bounded sample;
* redistribution -- the device redistribution program (one launch), us/call,
              next to the oracle port of the reference's sweep on one core.

``--impl reference`` times the reference CPU path (the oracle port of
reference_eval, multiprocess over host cores) on the same config and prints
its own line; ranks > 0 exit without work.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "images/sec of redistributed poly-CNN forward at 1 B200; % of roofline"
UNIT = "images/s"
L2_FLUSH_BYTES = 256 << 20


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# model preparation
# ---------------------------------------------------------------------------

def build_model(name: str):
    from paper_2509_22857_b200 import configs
    return configs.build(name)


def redistributed_engine(g, cfg, options=None):
    """Apply the config's redistribution on the device; return (engine, info)."""
    from paper_2509_22857_b200 import transforms as T
    from paper_2509_22857_b200.runtime import Engine
    eng = Engine(g, options=options)
    info = []
    cur = g
    for direction in cfg.redistribution:
        accepted, refused = T.plan_sweep(eng, cur, direction, allow_negative_leading=cfg.allow_negative_leading)
        prog = T.compile_sweep(eng, cur, direction, accepted, cfg.allow_negative_leading)
        T.run_program(eng, prog)
        info.append({"direction": direction, "donors": len(accepted), "refused": len(refused)})
        cur = eng.to_graph()
    return eng, cur, info


def time_redistribution(g, cfg, reps=20):
    """us per launch of the (last) sweep program, run in place on a scratch engine."""
    import torch
    from paper_2509_22857_b200 import transforms as T
    from paper_2509_22857_b200.runtime import Engine
    eng = Engine(g)
    direction = cfg.redistribution[0]
    accepted, _ = T.plan_sweep(eng, g, direction, allow_negative_leading=cfg.allow_negative_leading)
    prog = T.compile_sweep(eng, g, direction, accepted, cfg.allow_negative_leading)
    saved = eng.master.clone()
    times, dev_us, pack_us = [], [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for i in range(reps + 3):
        eng.master.copy_(saved)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T.run_program_on(eng.master, prog, eng.device, events=(ev[0], ev[1]))  # status read-back included
        eng.repack()
        ev[2].record()
        torch.cuda.synchronize()
        if i >= 3:
            times.append(time.perf_counter() - t0)
            dev_us.append(ev[0].elapsed_time(ev[1]) * 1e3)
            pack_us.append(ev[1].elapsed_time(ev[2]) * 1e3)
    return {"us_per_call": 1e6 * float(np.median(times)), "device_us": round(float(np.median(dev_us)), 1),
            "repack_device_us": round(float(np.median(pack_us)), 1), "direction": direction,
            "donors": len(accepted), "ops": len(prog.ops), "rewrites": len(prog.rewrite_descs()),
            "note": "us_per_call: wall time of pcnn_redistribute (one cooperative launch) + status read + repack; "
                    "device_us: CUDA events around the launch; repack_device_us: status read to repack end"}


# ---------------------------------------------------------------------------
# roofline bookkeeping, from the device timeline of graph replays
# ---------------------------------------------------------------------------

KERNEL_NAMES = {1: "conv_simt_kernel", 2: "conv_tc_kernel (3xTF32, A in TMEM)",
                3: "conv_tc_kernel (fp16x2, A in TMEM)", 5: "conv_ss_kernel (fp16x2, halo tiles in smem)",
                6: "conv_blk_kernel (fp16x2, image-resident runs)",
                7: "net_kernel (whole network in one launch, fp32 CUDA cores)"}
# fp32 FMA peak of the CUDA cores (148 SMs x 128 lanes x 2 FLOP x 1.965 GHz), the
# roofline of the whole-network kernel (derived from the SM count and max clock)
SIMT_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
OTHER_NAMES = {1: "ingest_kernel", 3: "linear_kernel", 12: "copyout_kernel"}
POOL_PASS = "pool pass behind a conv (localpool_kernel / bipool2_kernel)"


def unfused_stages(eng, plan, batch, ts, hbm_gbs):
    """North star: 'achieved HBM GB/s for unfused elementwise and pooling
    stages, each against B200 peak'.  Every launch of the timed plan that is
    not a tensor-core conv -- the NCHW ingest, a pooling pass behind a pooled
    conv (conv into a float32 scratch map, then the pool launch), standalone
    pool / elementwise units, dense layers -- with its algorithmic bytes
    (float32 input read once + output written once [+ weights]; the ingest's
    and the pools' split fp16 hi/lo outputs are 4 bytes per element too), its
    in-graph device time (Plan.timeline_passes) and the fraction of the
    measured HBM peak that makes."""
    lw = eng.lw
    n = plan.n_units
    um, pm = ts.unit_ms(), ts.pass_ms()

    def numel(t):
        d = lw.tensors[t]
        return batch * d.c * d.h * d.w

    rows = []
    for i, u in enumerate(lw.units):
        kind = u["kind"]
        if plan.unit_impl(i) == 7:
            continue
        if kind == 2:
            if pm[i] > 0:
                # the conv wrote its unpooled map; the pass reads it and writes the unit's output
                g, shapes = lw.graph, lw.shapes
                from paper_2509_22857_b200.graph import ConvNode
                conv = next(nid for nid in lw.unit_nodes[i] if isinstance(g.nodes[nid], ConvNode))
                co, ho, wo = shapes[conv]
                byts = 4.0 * (batch * co * ho * wo + numel(u["out"]))
                rows.append(("pool pass of unit %d" % i, pm[i], byts))
            continue
        if um[i] <= 0 or kind == 12:
            continue
        if kind == 3:
            byts = 4.0 * (batch * u["cin"] + batch * u["cout"] + u["cin"] * u["cout"] + u["cout"])
            name = "linear_kernel (unit %d)" % i
        else:
            byts = 4.0 * ((numel(u["in_"]) if u.get("in_", -1) >= 0 else numel(u["out"])) + numel(u["out"]))
            name = "%s (unit %d)" % (OTHER_NAMES.get(kind, "eltwise / pool kernel"), i)
        rows.append((name, um[i], byts))
    return [{"stage": nm, "us": round(ms * 1e3, 2), "algorithmic_bytes": int(b),
             "achieved_gbs": round(b / (ms * 1e-3) / 1e9, 1), "frac_hbm": round(b / (ms * 1e-3) / 1e9 / hbm_gbs, 3)}
            for nm, ms, b in rows]


def unit_cost(eng, i, batch):
    """(algorithmic FLOPs, algorithmic bytes) of conv unit i, from the graph's
    conv node (the reference's layer, not its lowered form -- e.g. RN18's
    7x7/s2 stem counts K = 3*7*7 = 147, not the space-to-depth K = 192):
    FLOP = 2 M N K, M = B Ho Wo, N = C_out, K = C_in kh kw; bytes = 4 (input
    once + output after the fused pool + residual + weights + bias)."""
    from paper_2509_22857_b200.graph import ConvNode
    lw = eng.lw
    g = lw.graph
    shapes = lw.shapes
    u = lw.units[i]
    conv = next(nid for nid in lw.unit_nodes[i] if isinstance(g.nodes[nid], ConvNode))
    node = g.nodes[conv]
    src = g.inputs_of(conv)[0]
    cin, h, w = shapes[src]
    cout, _, kh, kw = node.weight.shape
    ho, wo = shapes[conv][1], shapes[conv][2]
    m = batch * ho * wo
    flops = 2.0 * m * cout * cin * kh * kw
    out = 1
    for d in shapes[lw.unit_nodes[i][-1]]:
        out *= d
    byts = 4.0 * (batch * cin * h * w + batch * out + cout * cin * kh * kw + cout)
    if u.get("residual", 0):
        byts += 4.0 * batch * cout * ho * wo
    return flops, byts


def unit_family(eng, plan, i):
    u = eng.lw.units[i]
    if plan.unit_impl(i) == 7:
        return KERNEL_NAMES[7]
    if u["kind"] == 2:
        return KERNEL_NAMES[plan.unit_impl(i)]
    return OTHER_NAMES.get(u["kind"], "eltwise / pool kernels")


def union_ns(iv):
    """Total length of the union of [s, e) intervals."""
    tot, cur_s, cur_e = 0, None, None
    for s, e in sorted(iv):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


class TimelineStats:
    """Per-step device timelines (pcnn_plan_timeline: %globaltimer at each
    launch's first CTA start past its dependency wait and last CTA exit),
    read after every timed step.  For each kernel family: the union of its
    launches' intervals per step, so a family's time can never exceed the
    step."""

    def __init__(self, eng, plan):
        self.eng, self.plan = eng, plan
        n = self.n = plan.n_units
        self.launch_of = [plan.unit_launch(i) for i in range(n)]
        self.family = [unit_family(eng, plan, self.launch_of[i]) for i in range(n)]
        # rows n + u of Plan.timeline_passes: the pooling pass behind pooled conv unit u
        self.family += [POOL_PASS] * n
        self.fam_ns = {}
        self.unit_ns = np.zeros(2 * n)
        self.span_ns = []
        self.steps = 0

    def add(self, tl):
        live = [(i, int(s), int(e)) for i, (s, e) in enumerate(tl) if e > 0 and s > 0]
        if not live:
            return
        self.steps += 1
        self.span_ns.append(max(e for _, _, e in live) - min(s for _, s, _ in live))
        fams = {}
        for i, s, e in live:
            fams.setdefault(self.family[i], []).append((s, e))
            self.unit_ns[i] += e - s
        for f, iv in fams.items():
            self.fam_ns[f] = self.fam_ns.get(f, 0) + union_ns(iv)

    def family_ms(self):
        return {f: t / self.steps * 1e-6 for f, t in self.fam_ns.items()}

    def unit_ms(self):
        return self.unit_ns[:self.n] / max(self.steps, 1) * 1e-6

    def pass_ms(self):
        return self.unit_ns[self.n:] / max(self.steps, 1) * 1e-6

    def launches(self, fam):
        return sum(1 for i in range(self.n) if self.family[i] == fam and self.launch_of[i] == i
                   and (self.eng.lw.units[i]["kind"] == 2 or fam == KERNEL_NAMES[7]))


def roofline(eng, plan, batch, ts: TimelineStats, ms_per_step, config):
    """The dominant kernel family (largest share of the device-timed step):
    achieved = its algorithmic FLOPs (or bytes) per step / its graph-replay
    time per step (timeline union), against the fp32-accurate tensor rate of
    that kernel (three fp16 products at the dense fp16 = bf16 rate for the
    fp16x2 kernels: bf16/3; 3xTF32: bf16/6) or HBM bandwidth, whichever the
    per-layer roofline max(F/P, B/BW) says binds.  Also the SURVEY 8(d) step
    figure sum_l max(F_l/P, B_l/BW) / ms_per_step."""
    hbm, bf16, _, basis = peaks()
    rate = {3: bf16 / 3.0, 5: bf16 / 3.0, 6: bf16 / 3.0, 2: bf16 / 6.0, 1: bf16 / 6.0, 7: SIMT_FP32_TFLOPS}
    lw = eng.lw
    if not ts.steps:
        return {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                "note": "plan created without options.timeline: no device timeline"}
    fam_ms = ts.family_ms()
    dom = max(fam_ms, key=fam_ms.get)
    F = B = t_tensor = t_hbm = 0.0
    step_roof = 0.0
    per_layer = []
    for i, u in enumerate(lw.units):
        if u.get("kind") != 2:
            continue
        impl = plan.unit_impl(i)
        f, b = unit_cost(eng, i, batch)
        tl = max(f / (rate[impl] * 1e12), b / (hbm * 1e9))
        step_roof += tl
        if ts.family[i] == dom:
            F += f
            B += b
            t_tensor += f / (rate[impl] * 1e12)
            t_hbm += b / (hbm * 1e9)
        per_layer.append(round(tl * 1e6, 2))
    Tk = fam_ms[dom] * 1e-3
    P = rate[5] if "fp16x2" in dom else (rate[7] if dom == KERNEL_NAMES[7] else rate[2])
    bound = "tensor" if t_tensor >= t_hbm else "hbm"
    if bound == "tensor":
        achieved, peak, unit = F / Tk / 1e12, P, "TFLOP/s"
    else:
        achieved, peak, unit = B / Tk / 1e9, hbm, "GB/s"
    n = ts.launches(dom)
    ncu = measured_ncu(config)
    return {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": unit,
            "frac": round(achieved / peak, 4),
            "traffic": (ncu or {}).get("dram_bytes_per_launch"),
            "kernel": dom, "launches_per_step": n,
            "kernel_ms_per_step": round(fam_ms[dom], 4),
            "share_of_step": round(fam_ms[dom] / ms_per_step, 4),
            "frac_tensor": round(F / Tk / 1e12 / P, 4), "frac_hbm": round(B / Tk / 1e9 / hbm, 4),
            "algorithmic_per_launch": {"flops": F / max(n, 1), "bytes": B / max(n, 1)},
            "timing": "device timeline of every timed graph replay (pcnn_plan_timeline), union of the "
                      "family's launch intervals per step",
            "peak_basis": f"{basis} bf16_tflops {bf16} (tensor: /3 for fp16x2, /6 for 3xTF32); hbm_gbs {hbm}"
                          + (f"; fp32 CUDA-core FMA peak {SIMT_FP32_TFLOPS:.1f} (derived)" if dom == KERNEL_NAMES[7] else ""),
            "ncu": ncu,
            "note": ("image-resident runs: the bytes term above counts every layer's input and output once "
                     "(SURVEY 8d), but the run keeps intermediate tensors in shared memory -- ncu DRAM traffic per "
                     "launch is 'traffic'; frac_tensor is the binding measure for this family")
            if dom == KERNEL_NAMES[6] else None,
            "step": {"roofline_time_us": round(step_roof * 1e6, 1), "frac": round(step_roof * 1e3 / ms_per_step, 4),
                     "formula": "sum over conv layers of max(FLOP/P_kernel, bytes/BW) / measured ms_per_step"},
            "families_ms_per_step": {k: round(v, 4) for k, v in sorted(fam_ms.items(), key=lambda kv: -kv[1])}}


def measured_ncu(config):
    """ncu evidence for the dominant kernel from the committed capture
    summary (profiles/ncu_summary.json, tools/summarize_profiles.py)."""
    path = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(path.read_text()).get(config)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of levnet.graph.reference_eval
# ---------------------------------------------------------------------------

_POOL_G = None


def _worker_init(path):
    global _POOL_G
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_2509_22857_b200.graph import load_model
    _POOL_G = load_model(path)


def _worker_eval(x):
    from oracle import levnet_oracle as O
    return O.reference_eval(_POOL_G, x)


class CpuReference:
    """The float64 oracle over host cores: one process per core, each running
    reference_eval on whole images (OpenBLAS single-threaded per process)."""

    def __init__(self, g, procs: int | None = None):
        import multiprocessing as mp
        import tempfile
        from paper_2509_22857_b200.graph import save_model
        self.procs = procs or os.cpu_count() or 1
        self.tmp = tempfile.TemporaryDirectory()
        path = os.path.join(self.tmp.name, "m.json")
        save_model(g, path)
        env_before = os.environ.get("OPENBLAS_NUM_THREADS")
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_worker_init, initargs=(path,))
        if env_before is None:
            os.environ.pop("OPENBLAS_NUM_THREADS", None)
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = env_before
        self.i = 0

    def run(self, x, budget_s: float):
        """Evaluate rounds of `procs` images until budget_s elapses; (img/s, images, seconds)."""
        done, t0 = 0, time.perf_counter()
        while True:
            chunk = [x[(self.i + j) % len(x)] for j in range(self.procs)]
            self.pool.map(_worker_eval, chunk)
            self.i += len(chunk)
            done += len(chunk)
            el = time.perf_counter() - t0
            if el >= budget_s:
                return done / el, done, el

    def close(self):
        self.pool.terminate()
        self.tmp.cleanup()


def cpu_reference(g, x, budget_s: float):
    ref = CpuReference(g)
    try:
        ref.run(x[:1], 0.0)  # warm-up: imports and first touch in every worker
        ips, done, el = ref.run(x, budget_s)
    finally:
        ref.close()
    return ips, done, el, ref.procs


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def dist_env():
    from paper_2509_22857_b200.replicas import dist_env as env
    return env()


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2509_22857_b200 import configs
    cfg = configs.CONFIGS[args.config]
    g = build_model(args.config)
    x = configs.make_input(cfg, batch=min(cfg.batch, 64))
    ref = CpuReference(g)
    procs = ref.procs
    budget = max(0.5, min(6.0, 150.0 / max(args.steps + args.warmup, 1)))
    total_imgs, t = 0, 0.0
    try:
        for i in range(args.warmup + args.steps):
            _, done, el = ref.run(x, budget if i >= args.warmup else 0.0)
            if i >= args.warmup:
                total_imgs += done
                t += el
    finally:
        ref.close()
    value = total_imgs / t
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config}_b{cfg.batch}_forward", "global_batch": cfg.batch,
                       "note": "each step = a bounded sample of the batch's images"},
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{total_imgs} images of {args.config} over {args.steps} steps, "
                                       f"oracle reference_eval (float64, per image, levnet graph.py:413) "
                                       f"in {procs} processes"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def oracle_logits(gr, x_host):
    """float64 oracle forward of every image over the host cores (oracle/pool.py)."""
    from oracle.pool import OraclePool
    with OraclePool(gr) as pool:
        return pool.eval(x_host)


def precision_table(gr, x_host, want, flush, steps=5):
    """The same redistributed graph and batch under each arithmetic scheme the
    library has: device ms per forward (CUDA events, L2 flushed, graph replay)
    and max relative error of the logits against the float64 oracle on every
    image.  Rows: the default fp16x2 fast path (three fp16 products, fp32
    accumulation), forced 3xTF32 (kind::tf32, A from TMEM), the all-float32
    tensor plan (the rerun target when an activation leaves the fp16 range)
    and plain fp32 FFMA (conv_simt_kernel)."""
    import torch
    from paper_2509_22857_b200 import _lib as L
    from paper_2509_22857_b200.runtime import Engine
    x = torch.from_numpy(x_host).cuda()
    rows = []
    for label, impl in (("fp16x2 (default plan)", L.IMPL_AUTO), ("3xTF32 forced", L.IMPL_TF32),
                        ("float32 tensors (3xTF32 / SIMT)", L.IMPL_FP32_TENSORS), ("fp32 FFMA (SIMT)", L.IMPL_SIMT)):
        row = {"scheme": label, "impl": impl}
        try:
            eng = Engine(gr, impl=impl)
            out = torch.empty(eng.out_shape(len(x_host)), dtype=torch.float32, device="cuda")
            eng.forward(x, out)
            for _ in range(3):
                eng.forward(x, out, check=False)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            stream = torch.cuda.current_stream()
            for a, b in ev:
                flush()
                a.record(stream)
                eng.forward(x, out, check=False)
                b.record(stream)
            torch.cuda.synchronize()
            y = out.cpu().numpy().reshape(want.shape).astype(np.float64)
            plan = eng.plan(len(x_host))
            row.update({"ms_per_step": round(sum(a.elapsed_time(b) for a, b in ev) / steps, 4),
                        "max_rel_err": float(np.max(np.abs(y - want)) / max(float(np.max(np.abs(want))), 1e-30)),
                        "allclose_rtol1e-4_atol1e-5": bool(np.allclose(y, want, rtol=1e-4, atol=1e-5)),
                        "fp32_reruns": int(eng.fallbacks),
                        "conv_impl": sorted({plan.unit_impl(i) for i, u in enumerate(eng.lw.units)
                                             if u.get("kind") == 2})})
            del eng, out
            torch.cuda.empty_cache()
        except Exception as e:  # a scheme a shape class does not support is reported, not hidden
            row["error"] = f"{type(e).__name__}: {e}"[:200]
        rows.append(row)
    return rows


def parity_of(gr, x_host, y, want=None):
    """Max relative error of the timed batch's logits against the float64
    oracle forward of the same (redistributed) graph, every image, over the
    host cores (oracle/pool.py) -- the checker, not the measured path."""
    t0 = time.perf_counter()
    if want is None:
        want = oracle_logits(gr, x_host)
    y = y.reshape(want.shape).astype(np.float64)
    err = float(np.max(np.abs(y - want)) / max(float(np.max(np.abs(want))), 1e-30))
    cy, cw = y - y.mean(0), want - want.mean(0)
    cerr = float(np.max(np.abs(cy - cw)) / max(float(np.max(np.abs(cw))), 1e-30))
    close = bool(np.allclose(y, want, rtol=1e-4, atol=1e-5))
    return {"max_rel_err": err, "centred_rel_err": cerr, "allclose_rtol1e-4_atol1e-5": close,
            "images": int(len(x_host)), "argmax_agree": float(np.mean(np.argmax(y, 1) == np.argmax(want, 1))),
            "vs": "float64 oracle reference_eval restatement of the redistributed graph, every image of the "
                  "timed batch", "oracle_s": round(time.perf_counter() - t0, 2)}


def measure(name, args, rank, world, local, flush, options, e2e=True):
    """Time one config's redistributed forward; returns the pieces of a line."""
    import torch
    from paper_2509_22857_b200 import configs, replicas
    cfg = configs.CONFIGS[name]
    batch = (args.batch or cfg.batch) if name == args.config else cfg.batch
    g = build_model(name)
    eng, gr, redist_info = redistributed_engine(g, cfg, options)
    x_host = configs.make_input(cfg, batch=batch, seed=2 + rank).astype(np.float32)
    x = torch.from_numpy(x_host).cuda()
    out = torch.empty(eng.out_shape(batch), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    # one checked forward: if an activation overflows the fp16 split format the
    # engine reruns it in float32 and rescales those tensors (Engine.recalibrate)
    eng.forward(x, out)
    for _ in range(max(args.warmup, 3)):
        eng.forward(x, out, check=False)
    plan = eng.plan(batch)
    ts = TimelineStats(eng, plan)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        # keep the GPU under the same load while the sampler spins up, so the
        # clock samples bracket the timed steps (which can be only ~ms long)
        t_end = time.perf_counter() + 0.6
        while time.perf_counter() < t_end:
            flush()
            eng.forward(x, out, check=False)
            torch.cuda.synchronize()
        for i in range(args.steps):
            flush()
            starts[i].record(stream)
            eng.forward(x, out, check=False)
            ends[i].record(stream)
            # the step's launch timeline (D2H after its end event; not timed)
            if options.timeline:
                ts.add(plan.timeline_passes())
        torch.cuda.synchronize()
        t_end = time.perf_counter() + 0.3
        while time.perf_counter() < t_end:
            flush()
            eng.forward(x, out, check=False)
            torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms = replicas.max_over_ranks(ms)
    res = {"name": name, "cfg": cfg, "batch": batch, "g": g, "gr": gr, "eng": eng, "plan": plan, "ts": ts,
           "x_host": x_host, "out": out, "ms": ms, "clocks": clocks.summary(), "redist_info": redist_info,
           "value": world * batch * args.steps / (ms * 1e-3)}
    # fp16x2 fast path valid only if no split-format activation left the fp16 range
    assert plan.status() == 0, "fp16 range overflow: result needs the fp32 rerun"
    assert np.all(np.isfinite(out.cpu().numpy())), "non-finite logits"
    if not e2e:
        return res

    # e2e through the C ABI with pinned host buffers
    xh = torch.from_numpy(x_host).pin_memory()
    oh = torch.empty(eng.out_shape(batch), dtype=torch.float32).pin_memory()
    xd = torch.empty_like(x)
    od = torch.empty_like(out)
    from paper_2509_22857_b200 import _lib as L
    import ctypes
    from paper_2509_22857_b200.runtime import _stream_handle

    def e2e_step():
        L.check(L.lib().pcnn_forward_host(plan.handle, ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(oh.data_ptr()),
                                          ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(od.data_ptr()),
                                          _stream_handle()), "pcnn_forward_host")

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    e_ms = 0.0
    for i in range(args.steps):
        flush()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        e2e_step()
        s1.record(stream)
        torch.cuda.synchronize()
        e_ms += s0.elapsed_time(s1)
    e_ms = replicas.max_over_ranks(e_ms)
    res["e2e_serial"] = world * batch * args.steps / (e_ms * 1e-3)

    # e2e, pipelined: the same K steps through Engine.forward_host_many
    # (pcnn_forward_host_many) -- every step still copies its input in and
    # its logits out, but step i+1's H2D overlaps step i's forward
    outs_h = [torch.empty(eng.out_shape(batch), dtype=torch.float32).pin_memory() for _ in range(args.steps)]
    staging = (xd, torch.empty_like(x), od)
    for _ in range(2):
        eng.forward_host_many([xh] * 3, outs_h[:3], staging=staging)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush()
    p0.record(stream)
    eng.forward_host_many([xh] * args.steps, outs_h, staging=staging, sync=False)
    p1.record(stream)
    torch.cuda.synchronize()
    p_ms = replicas.max_over_ranks(p0.elapsed_time(p1))
    res["e2e"] = world * batch * args.steps / (p_ms * 1e-3)
    ref = out.cpu().numpy()
    for o in outs_h:
        np.testing.assert_allclose(o.numpy(), ref, rtol=1e-5, atol=1e-6)
    # fused global pools reduce with float atomics, so repeated runs agree to rounding only
    np.testing.assert_allclose(oh.numpy(), ref, rtol=1e-5, atol=1e-6)
    assert plan.last_status() == 0, "fp16 range overflow: result needs the fp32 rerun"
    any_split = any(plan.tensor_split(t) for t in range(len(eng.lw.tensors)))
    res["h2d"] = int(xh.numel() * 4)
    res["d2h"] = int(oh.numel() * 4) + (4 if any_split else 0)
    return res


def record(res, args, world):
    """The per-config fields of the JSON line."""
    eng, plan, batch, ms = res["eng"], res["plan"], res["batch"], res["ms"]
    ms_step = ms / args.steps
    roof = roofline(eng, plan, batch, res["ts"], ms_step, res["name"])
    cfg = res["cfg"]
    rec = {"value": round(res["value"], 2), "ms_per_step": round(ms_step, 4),
           "config": {"workload": f"{res['name']}_b{batch}_redistributed_forward", "model": res["name"],
                      "global_batch": batch * world, "input": "x".join(map(str, cfg.input_shape)),
                      "parallelism": f"replicas{world}", "l2": "flushed (256 MiB write) between timed steps",
                      "redistribution": res["redist_info"],
                      "conv_impl": sorted({plan.unit_impl(i) for i, u in enumerate(eng.lw.units)
                                           if u.get("kind") == 2}),
                      "split_tensors": sum(plan.tensor_split(t) > 0 for t in range(len(eng.lw.tensors)))},
           "gpu_launches": plan.launches() * args.steps,
           "roofline": roof, "clocks": res["clocks"],
           "device_step_span_ms": round(float(np.median(res["ts"].span_ns)) * 1e-6, 4) if res["ts"].steps else None,
           "unit_ms": [round(float(v), 4) for v in res["ts"].unit_ms()]}
    if res["ts"].steps:
        rec["unfused_stages"] = unfused_stages(eng, plan, batch, res["ts"], peaks()[0])
    if "e2e" in res:
        rec["e2e"] = {"value": round(res["e2e"], 2), "unit": UNIT, "h2d_bytes_per_step": res["h2d"],
                      "d2h_bytes_per_step": res["d2h"],
                      "api": "Engine.forward_host_many -> pcnn_forward_host_many (pinned host batches, "
                             "H2D of step i+1 overlapping step i; no L2 flush inside the pipeline)",
                      "serial_value": round(res["e2e_serial"], 2),
                      "serial_api": "pcnn_forward_host per step (H2D, forward, D2H, sync; L2 flushed between steps)"}
    return rec


def time_cpu_redistribution(g, cfg, budget_s=2.0):
    """The oracle port of the reference's per-donor sweeps (transforms.py:
    423-485, float64 on one host core) for the same config: ms per call."""
    from oracle import levnet_oracle as O
    times = []
    t_end = time.perf_counter() + budget_s
    while not times or (time.perf_counter() < t_end and len(times) < 20):
        t0 = time.perf_counter()
        cur = g
        for d in cfg.redistribution:
            cur, _, _ = O.redistribute_sweep(cur, d, allow_negative_leading=cfg.allow_negative_leading)
        times.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(times)), len(times)


def run_ours(args):
    import torch
    from paper_2509_22857_b200 import replicas
    from paper_2509_22857_b200 import _lib as L
    rank, world, local = dist_env()
    if world > 1:
        replicas.init_replicas("nccl")  # replicas only: the group carries the barrier and max-over-ranks
    else:
        torch.cuda.set_device(0)
    from paper_2509_22857_b200 import configs
    L.require_device()
    # default plan options; PCNN_* developer variables (tools/, profiling) are
    # applied here explicitly and recorded in the line when they change anything
    options = L.options_from_env()
    flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def flush():
        flush_buf.fill_(1.0)

    main = measure(args.config, args, rank, world, local, flush, options)
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    rec = record(main, args, world)
    line = {"metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic"}
    line.update({k: v for k, v in rec.items() if k not in ("value", "ms_per_step")})
    default = L.PlanOptions.default().as_dict()
    changed = {k: v for k, v in options.as_dict().items() if default.get(k) != v}
    if changed:
        line["config"]["plan_options"] = changed
    cfg = main["cfg"]
    # every timed measurement first (main, then secondary configs); the
    # checkers and CPU work afterwards, so their host processes never overlap
    # a timed region
    secondary = [c for c in args.secondary.split(",") if c and c != args.config] if world == 1 else []
    checks = [(line, main["gr"], main["x_host"], main["out"].cpu().numpy())]
    main_g = main["g"]
    del main
    torch.cuda.empty_cache()
    if secondary:
        line["secondary"] = {}
        for name in secondary:
            res = measure(name, args, rank, world, local, flush, options, e2e=True)
            sub = record(res, args, world)
            sub["metric"] = METRIC
            sub["unit"] = UNIT
            line["secondary"][name] = sub
            checks.append((sub, res["gr"], res["x_host"], res["out"].cpu().numpy()))
            del res
            torch.cuda.empty_cache()
    if not args.no_parity:
        for dst, gr, xh, y in checks:
            t0 = time.perf_counter()
            want = oracle_logits(gr, xh)
            oracle_s = round(time.perf_counter() - t0, 2)
            dst["parity"] = parity_of(gr, xh, y, want)
            dst["parity"]["oracle_s"] = oracle_s
            if not args.no_precision and world == 1:
                dst["precision"] = precision_table(gr, xh, want, flush)
    if not args.no_redist_timing:
        red = time_redistribution(main_g, cfg)
        cpu_ms, n = time_cpu_redistribution(main_g, cfg)
        red["cpu_reference_ms_per_call"] = round(cpu_ms, 3)
        red["cpu_reference"] = (f"oracle port of levnet redistribute_{'/'.join(cfg.redistribution)} per-donor "
                                f"sweep (transforms.py:423-485), float64, 1 host core, median of {n}")
        line["redistribution"] = red
    if not args.no_cpu and world == 1:
        g = build_model(args.config)
        ips, done, el, procs = cpu_reference(g, configs.make_input(cfg, batch=64), args.cpu_seconds)
        line["cpu_baseline"] = {"value": round(ips, 3), "unit": UNIT, "cores": procs, "kind": "port",
                                "sample": f"{done} images in {el:.1f} s, float64 oracle reference_eval "
                                          f"(restates levnet graph.py:413) in {procs} processes"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="resnet20")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-redist-timing", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-precision", action="store_true",
                    help="skip the per-scheme precision / time table (fp16x2, 3xTF32, float32 tensors, SIMT)")
    ap.add_argument("--secondary", default="resnet18",
                    help="comma-separated configs measured after the main one (1 GPU), reported under 'secondary'")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
