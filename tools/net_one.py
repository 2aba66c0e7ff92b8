"""One LeNet forward on the whole-network kernel (for ncu)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs, _lib as L, transforms as T
from paper_2509_22857_b200.runtime import Engine
cfg = configs.CONFIGS["lenet5"]
g = configs.build("lenet5")
for d in cfg.redistribution:
    g, _, _ = T.redistribute_sweep(g, d)
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = torch.from_numpy(configs.make_input(cfg, batch=batch).astype(np.float32)).cuda()
eng = Engine(g, options=L.PlanOptions.default(graph=0))
for _ in range(3):
    eng.forward(x, check=False)
torch.cuda.synchronize()
