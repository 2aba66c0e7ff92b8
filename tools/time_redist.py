"""Breakdown of one device redistribution sweep: the pcnn_redistribute launch
(+ status read) and the repack (pcnn_pack), CUDA events and wall clock."""
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200 import transforms as T
from paper_2509_22857_b200.runtime import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
cfg = configs.CONFIGS[name]
g = configs.build(name)
eng = Engine(g, options=_L.options_from_env())
direction = cfg.redistribution[0]
accepted, _ = T.plan_sweep(eng, g, direction, allow_negative_leading=cfg.allow_negative_leading)
prog = T.compile_sweep(eng, g, direction, accepted, cfg.allow_negative_leading)
saved = eng.master.clone()
rows = []
for i in range(13):
    eng.master.copy_(saved)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    T.run_program(eng, prog)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng.repack()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if i >= 3:
        rows.append((t1 - t0, t2 - t1))
r = np.median(np.array(rows), axis=0) * 1e6
print(f"{name}: run_program (launch + status read + repack) {r[0]:.0f} us, repack alone {r[1]:.0f} us, "
      f"ops {len(prog.ops)}, pack ops {len(eng.lw.pack_ops)}")
