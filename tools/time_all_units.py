"""Device-timeline time of EVERY unit of a config under several plan option
sets (A/B experiments): python tools/time_all_units.py resnet18 'debug=2' 'debug=4'"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs, _lib as L
from paper_2509_22857_b200.runtime import Engine
name = sys.argv[1]
cfg = configs.CONFIGS[name]
g = configs.build(name)
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
for spec in ["default"] + sys.argv[2:]:
    kw = {} if spec == "default" else {k: type(getattr(L.PlanOptions.default(), k))(v) for k, v in
                                       (p.split("=") for p in spec.split(","))}
    eng = Engine(g, options=L.PlanOptions.default(**kw))
    for _ in range(3):
        eng.forward(x, check=False)
    plan = eng.plan(cfg.batch)
    ts, gs, spans = [], [], []
    for _ in range(10):
        eng.forward(x, check=False)
        tl = plan.timeline()
        ts.append((tl[:, 1] - tl[:, 0]) * 1e-3)
        on = tl[tl[:, 0] > 0]
        gs.append((on[1:, 0] - on[:-1, 1]) * 1e-3)
        spans.append((on[-1, 1] - on[0, 0]) * 1e-3)
    t = np.median(np.array(ts), axis=0)
    gap = np.median(np.array(gs), axis=0)
    print(f"{spec:24s} total {t.sum():8.1f} us span {np.median(spans):7.1f} | " + " ".join(f"{i}:{v:.1f}" for i, v in enumerate(t) if v > 0))
    print(f"{'':24s} gaps  " + " ".join(f"{v:.1f}" for v in gap))
