"""Compare every unit's output tensor (whole batch) between two plans of one
config: the default and one built with an env switch set (e.g.
PCNN_NO_STREAMK=1).  python tools/cmp_plans.py resnet18 PCNN_NO_STREAMK=1"""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs, transforms as T
from paper_2509_22857_b200.runtime import Engine
name = sys.argv[1]
k, v = sys.argv[2].split("=")
cfg = configs.CONFIGS[name]
g = configs.build(name)
for d in cfg.redistribution:
    g, _, _ = T.redistribute_sweep(g, d, allow_negative_leading=cfg.allow_negative_leading)
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
from paper_2509_22857_b200 import _lib as _L
ea = Engine(g); ya = ea.forward(x).cpu().numpy(); pa = ea.plan(cfg.batch)
os.environ[k] = v
eb = Engine(g, options=_L.options_from_env()); yb = eb.forward(x).cpu().numpy(); pb = eb.plan(cfg.batch)
print("logits max rel diff", float(np.abs(ya - yb).max() / np.abs(yb).max()))
for i, u in enumerate(ea.lw.units):
    t = u.get("out", -1)
    if t is None or t < 0:
        continue
    a, b = pa.read_tensor(t), pb.read_tensor(t)
    d = np.abs(a - b).reshape(a.shape[0], -1).max(1) / max(np.abs(b).max(), 1e-30)
    bad = np.nonzero(d > 1e-4)[0]
    print(f"unit {i:2d} kind {u['kind']} impl {pa.unit_impl(i)} max rel {d.max():.2e} bad images {bad[:12].tolist()} n_bad {len(bad)}")
