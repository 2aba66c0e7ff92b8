"""Device-timeline time of one unit of a config under several plan option
sets (A/B experiments): python tools/time_unit_opts.py resnet18 1 'debug=4096' 'debug=8192'"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs, _lib as L
from paper_2509_22857_b200.runtime import Engine
name, unit = sys.argv[1], int(sys.argv[2])
cfg = configs.CONFIGS[name]
g = configs.build(name)
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
for spec in ["default"] + sys.argv[3:]:
    kw = {} if spec == "default" else {k: type(getattr(L.PlanOptions.default(), k))(v) for k, v in
                                       (p.split("=") for p in spec.split(","))}
    eng = Engine(g, options=L.PlanOptions.default(**kw))
    for _ in range(3):
        eng.forward(x, check=False)
    plan = eng.plan(cfg.batch)
    ts = []
    for _ in range(10):
        eng.forward(x, check=False)
        tl = plan.timeline()
        ts.append((tl[unit, 1] - tl[unit, 0]) * 1e-3)
    tot = []
    print(f"{spec:30s} unit {unit}: {np.median(ts):8.2f} us")
