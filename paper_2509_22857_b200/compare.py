"""GPU verification report: the hot-path part of levnet's ``compare`` command
(reference cli.py:554-629) on the B200 engine.

The reference's ``compare`` runs three checks: transform equivalence
(``check_equivalence``, transforms.py:753-778, 100 float64 forwards of each
model, one image at a time), the FHE level table and the slot-simulator
fidelity.  The last two belong to the FHE planner / simulator, which this
build does not cover.  This module keeps the first and
adds what a batched GPU forward makes cheap:

* ``transform-equivalence`` -- the same metric and inputs as
  check_equivalence (U(-1, 1) draws from default_rng(seed), max|a-b| /
  max|a| per input, worst over inputs, argmax agreement), over 1000 inputs
  by default, both models streamed through ``Engine.forward_host_many``
  (host batches in, logits out, copies overlapping forwards);
* ``precision`` -- per fused unit of the transformed model, the largest
  deviation of its output tensor (read back with ``Plan.read_tensor``) on
  the fast path (fp16x2 tensor cores over split activations) from the same
  unit on float32 tensors (3xTF32 / SIMT), relative to that tensor's max:
  where in the network the three-product scheme loses accuracy, if
  anywhere.

    python -m paper_2509_22857_b200.compare --config resnet20 [--strategy forward]
    python -m paper_2509_22857_b200.compare --model m.json --strategy P2FR --json report.json
    python -m paper_2509_22857_b200.compare --model m.json --compiled t.json

Exit status 0 if every check passes, 1 otherwise (the reference raises
CheckFailure, exit 1).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from typing import Dict, Optional

import numpy as np

from . import _lib as L
from .graph import ModelGraph, load_model
from .runtime import Engine
from .transforms import DEVICE_RTOL, apply_pipeline, redistribute_sweep

FORMAT_NAMES = {0: "float32", 1: "split fp16 hi/lo", 2: "split fp16 hi/lo, parity planes"}


def _inputs(g: ModelGraph, n: int, seed: int) -> np.ndarray:
    """check_equivalence's inputs: one U(-1, 1) draw per input, in order."""
    shape = g.validate()[g.input_id()]
    rng = np.random.default_rng(seed)
    return np.stack([rng.uniform(-1.0, 1.0, shape) for _ in range(n)]).astype(np.float32)


def _stream(eng: Engine, xs: np.ndarray, batch: int) -> np.ndarray:
    """Logits of every input: full batches through forward_host_many, the
    remainder (if any) as one smaller batch."""
    import torch
    n = len(xs)
    full = n // batch
    outs = []
    if full:
        hb = [torch.from_numpy(xs[i * batch:(i + 1) * batch]).pin_memory() for i in range(full)]
        outs += [o.numpy().reshape(batch, -1) for o in eng.forward_host_many(hb)]
    if n % batch:
        outs.append(eng.forward_host(xs[full * batch:]).reshape(n % batch, -1))
    return np.concatenate(outs).astype(np.float64)


def equivalence_check(ref: ModelGraph, cand: ModelGraph, n_inputs: int = 1000, rtol: Optional[float] = None,
                      seed: int = 0, batch: int = 256) -> Dict:
    rtol = DEVICE_RTOL if rtol is None else rtol
    xs = _inputs(ref, n_inputs, seed)
    cand.validate()
    ea, eb = Engine(ref), Engine(cand)
    t0 = time.perf_counter()
    a = _stream(ea, xs, batch)
    b = _stream(eb, xs, batch)
    el = time.perf_counter() - t0
    err = np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(a), axis=1), 1e-12)
    worst = float(err.max())
    return {"name": "transform-equivalence", "passed": bool(worst <= rtol), "max_rel_err": worst,
            "argmax_match_rate": float(np.mean(np.argmax(a, 1) == np.argmax(b, 1))), "n_inputs": n_inputs,
            "rtol": rtol, "worst_input": int(err.argmax()),
            "forwards_per_s": round(2 * n_inputs / el, 1),
            "api": "Engine.forward_host_many (pinned host batches of %d)" % batch,
            "reference": "levnet check_equivalence transforms.py:753-778 / compare cli.py:554-629"}


def precision_check(g: ModelGraph, n_inputs: int = 64, seed: int = 0, tol: float = DEVICE_RTOL) -> Dict:
    """Per unit: fast-path output vs the float32-tensor plan's output."""
    import torch
    xs = torch.from_numpy(_inputs(g, n_inputs, seed + 1)).cuda()
    fast = Engine(g)
    ref = Engine(g, impl=L.IMPL_FP32_TENSORS, lowered=fast.lw)
    yf = fast.forward(xs).double().cpu().numpy()
    yr = ref.forward(xs).double().cpu().numpy()
    pf, pr = fast.plan(n_inputs), ref.plan(n_inputs)
    rows = []
    for i, (u, nodes) in enumerate(zip(fast.lw.units, fast.lw.unit_nodes)):
        t = u.get("out", -1)
        if t is None or t < 0 or u["kind"] in (L.UNIT_INGEST, L.UNIT_COPYOUT) or not pf.materialized(i):
            continue
        a, b = pf.read_tensor(t).astype(np.float64), pr.read_tensor(t).astype(np.float64)
        scale = max(float(np.abs(b).max()), 1e-30)
        rows.append({"unit": i, "nodes": nodes, "impl": pf.unit_impl(i),
                     "output_format": FORMAT_NAMES.get(pf.tensor_split(t), "?"),
                     "max_rel_err_vs_fp32": float(np.abs(a - b).max() / scale)})
    logits = float(np.abs(yf - yr).max() / max(float(np.abs(yr).max()), 1e-30))
    return {"name": "precision", "passed": bool(logits <= tol), "logits_max_rel_err_vs_fp32": logits, "tol": tol,
            "n_inputs": n_inputs, "fallbacks": fast.fallbacks, "units": rows,
            "note": "fast path = fp16x2 tensor cores on split activations; reference plan = float32 tensors "
                    "(3xTF32 / SIMT); errors relative to each tensor's max"}


def compare_report(reference: ModelGraph, transformed: ModelGraph, n_inputs: int = 1000,
                   rtol: Optional[float] = None, seed: int = 0, precision_inputs: int = 64) -> Dict:
    checks = [equivalence_check(reference, transformed, n_inputs, rtol, seed)]
    if precision_inputs:
        checks.append(precision_check(transformed, precision_inputs, seed))
    return {"passed": all(c["passed"] for c in checks), "checks": checks}


def _transform(g: ModelGraph, strategy: str, allow_negative_leading: bool = False) -> ModelGraph:
    s = strategy.lower()
    if s in ("forward", "backward"):
        out, _, _ = redistribute_sweep(g, s, allow_negative_leading=allow_negative_leading)
        return out
    out, _ = apply_pipeline(g, strategy.upper())
    return out


def main(argv=None) -> int:
    from . import configs
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--config", choices=sorted(configs.CONFIGS), help="a benchmark configuration")
    src.add_argument("--model", help="a neutral-format model file (graph.save_model / levnet export)")
    ap.add_argument("--strategy", default=None,
                    help="forward | backward (per-donor sweeps) | P2R | P2FR | P4 (apply_pipeline); "
                         "default: the config's own redistribution, else forward")
    ap.add_argument("--compiled", default=None, help="the transformed model as a file (skips the transform)")
    ap.add_argument("--n-inputs", type=int, default=1000)
    ap.add_argument("--equiv-rtol", type=float, default=None, help=f"default {DEVICE_RTOL} (float32 compute)")
    ap.add_argument("--precision-inputs", type=int, default=64, help="0 skips the per-unit precision check")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--json", dest="json_path", default=None)
    args = ap.parse_args(argv)
    L.require_device()
    if args.config:
        cfg = configs.CONFIGS[args.config]
        reference = configs.build(args.config)
        if args.compiled:
            transformed = load_model(args.compiled)
        elif args.strategy:
            transformed = _transform(reference, args.strategy, cfg.allow_negative_leading)
        else:
            transformed = reference
            for d in cfg.redistribution:
                transformed = _transform(transformed, d, cfg.allow_negative_leading)
    else:
        reference = load_model(args.model)
        transformed = load_model(args.compiled) if args.compiled else _transform(reference, args.strategy or "forward")
    payload = compare_report(reference, transformed, args.n_inputs, args.equiv_rtol, args.seed,
                             args.precision_inputs)
    text = json.dumps(payload, indent=2)
    if args.json_path:
        with open(args.json_path, "w") as fh:
            fh.write(text + "\n")
    print(text)
    if not payload["passed"]:
        first = next(c["name"] for c in payload["checks"] if not c["passed"])
        print(f"FAIL: {first} check failed", file=sys.stderr)
        return 1
    print("PASS")
    return 0


if __name__ == "__main__":
    sys.exit(main())
