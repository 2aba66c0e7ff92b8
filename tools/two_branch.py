"""Experiment: does splitting a batch into two concurrent graph replays (two
plans on two streams) hide the per-launch fill / drain overheads?

  python tools/two_branch.py resnet20 [splits]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200.runtime import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = configs.CONFIGS[name]
g = configs.build(name)
B = cfg.batch
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
engs = [Engine(g, options=_L.options_from_env()) for _ in range(ns)]
streams = [torch.cuda.Stream() for _ in range(ns)]
parts = [x[i * B // ns:(i + 1) * B // ns].contiguous() for i in range(ns)]
outs = [torch.empty(p.shape[0], 10 if cfg.name != "resnet18" else 1000, device="cuda") for p in parts]
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(fn, reps=20):
    ts = []
    for _ in range(reps + 3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[3:]))


full = Engine(g, options=_L.options_from_env())
out = torch.empty(B, outs[0].shape[1], device="cuda")
full.forward(x, out=out)
print("one plan, batch", B, "ms", round(timed(lambda: full.forward(x, out=out, check=False)), 4))
one = engs[0]
print("one plan, batch", B // ns, "ms", round(timed(lambda: one.forward(parts[0], out=outs[0], check=False)), 4))
for e, p, o in zip(engs, parts, outs):
    e.forward(p, out=o)


def conc():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    for e, p, o, s in zip(engs, parts, outs, streams):
        s.wait_event(ev)
        e.forward(p, out=o, stream=s, check=False)
    for s in streams:
        cur.wait_stream(s)


print(ns, "plans concurrent, batch", B, "ms", round(timed(conc), 4))
got = torch.cat(outs)
print("max |diff| vs one plan", float((got - out).abs().max()))
