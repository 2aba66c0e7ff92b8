"""In-graph launch timeline of one config: per launch start / end (us from the
first start) and the gap to the previous launch's end, median of N forwards
with the L2 flushed before each."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = configs.CONFIGS[name]
g = bench.build_model(name)
eng, gr, _ = bench.redistributed_engine(g, cfg, _L.options_from_env())
b = cfg.batch
x = torch.from_numpy(configs.make_input(cfg, batch=b, seed=2).astype(np.float32)).cuda()
out = torch.empty(eng.out_shape(b), dtype=torch.float32, device="cuda")
eng.forward(x, out)
plan = eng.plan(b)
fl = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
rows = []
for r in range(reps + 3):
    fl.fill_(1.0)
    eng.forward(x, out, check=False)
    t = plan.timeline().astype(np.float64)
    if r >= 3:
        rows.append(t)
T = np.stack(rows)  # reps, units, 2
live = [i for i in range(T.shape[1]) if T[0, i, 0] > 0]
t0 = T[:, live[0], 0][:, None]
st = np.median(T[:, live, 0] - t0, axis=0) / 1e3
en = np.median(T[:, live, 1] - t0, axis=0) / 1e3
prev = 0.0
print("unit  start    end     dur    gap(us)")
for k, i in enumerate(live):
    print("%3d %7.1f %7.1f %7.1f %6.1f" % (i, st[k], en[k], en[k] - st[k], st[k] - prev))
    prev = en[k]
print("span %.1f us" % en[-1])
