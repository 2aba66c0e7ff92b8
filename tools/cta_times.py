"""Per-launch CTA timeline of the halo-tile conv kernels inside one forward
(graph replay by default; PCNN_NO_GRAPH=1 for eager launches).

  PCNN_TC_DEBUG=64 python tools/cta_times.py resnet20

For each conv_ss launch (in execution order), relative to the first launch's
first CTA entry, in microseconds:
  entry   first CTA entry            (scheduling of the grid)
  wait    first/last griddepcontrol.wait return (previous grid complete)
  work    median CTA role-loop end   (t2)
  end     last CTA exit              (t3)
and the gap between one launch's last exit and the next launch's first wait
return (launch + dependency overhead)."""
import ctypes
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_22857_b200 import _lib as L
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200.runtime import Engine

assert int(os.environ.get("PCNN_TC_DEBUG", "0")) & 64, "set PCNN_TC_DEBUG=64"
name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
lib = L.lib()
fn = lib.pcnn_ss_cta_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
fn.restype = ctypes.c_int
SLOTS, CTAS = 64, 160
fn(None, 2)
cfg = configs.CONFIGS[name]
eng = Engine(configs.build(name), options=_L.options_from_env())
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
for _ in range(3):
    eng.forward(x, check=False)
torch.cuda.synchronize()
fn(None, 1)
eng.forward(x, check=False)
torch.cuda.synchronize()
buf = np.zeros((SLOTS, CTAS, 4), dtype=np.uint64)
fn(buf.ctypes.data, 0)
rows = []
for s in range(SLOTS):
    t = buf[s].astype(np.int64)
    live = t[:, 0] > 0
    if not live.any():
        continue
    t = t[live]
    rows.append((t[:, 0].min(), s, t))
rows.sort()
t00 = rows[0][0]
print(f"{name}: {len(rows)} conv_ss launches, times in us from the first CTA entry")
print(" # slot ctas   entry  wait0  wait1   work50  end    dur(wait0->end)  gap(prev end->wait0)")
prev_end = None
tot_gap = 0.0
for i, (_, s, t) in enumerate(rows):
    us = lambda v: (v - t00) / 1000.0
    e0, w0, w1 = us(t[:, 0].min()), us(t[:, 1].min()), us(t[:, 1].max())
    wk, en = us(np.median(t[:, 2])), us(t[:, 3].max())
    gap = (w0 - prev_end) if prev_end is not None else 0.0
    tot_gap += gap
    print(f"{i:2d} {s:4d} {len(t):4d} {e0:7.1f} {w0:6.1f} {w1:6.1f} {wk:8.1f} {en:6.1f} {en - w0:10.1f} {gap:12.1f}")
    prev_end = en
print(f"span {us(rows[-1][2][:, 3].max()):.1f} us, sum of gaps {tot_gap:.1f} us")
