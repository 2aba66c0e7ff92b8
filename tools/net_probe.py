"""Device time of LeNet's forward per plan variant (whole-network kernel vs layered)."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs, _lib as L, transforms as T
from paper_2509_22857_b200.runtime import Engine
cfg = configs.CONFIGS["lenet5"]
g = configs.build("lenet5")
for d in cfg.redistribution:
    g, _, _ = T.redistribute_sweep(g, d)
for batch in (1, 64, 512):
    x = torch.from_numpy(configs.make_input(cfg, batch=batch).astype(np.float32)).cuda()
    for net in (1, 0):
        eng = Engine(g, options=L.PlanOptions.default(fused_net=net))
        for _ in range(5):
            eng.forward(x, check=False)
        plan = eng.plan(batch)
        ts = []
        for _ in range(20):
            eng.forward(x, check=False)
            tl = plan.timeline()
            live = [(s, e) for s, e in tl if e > 0 and s > 0]
            ts.append((max(e for _, e in live) - min(s for s, _ in live)) * 1e-3)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(50):
            eng.forward(x, check=False)
        en.record(); torch.cuda.synchronize()
        print(f"batch {batch:4d} fused_net={net}: timeline span {np.median(ts):8.2f} us, events {st.elapsed_time(en) / 50 * 1e3:8.2f} us/forward, launches {plan.launches()}, impl {plan.unit_impl(1)}")
