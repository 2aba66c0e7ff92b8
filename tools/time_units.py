"""Per-unit CUDA-event times of one config (eager launches, warm)."""
import sys, pathlib, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200.runtime import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
impl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = configs.CONFIGS[name]
g = configs.build(name)
eng = Engine(g, impl=impl, options=_L.options_from_env())
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
out = eng.forward(x)
plan = eng.plan(x.shape[0])
n = plan.n_units
acc = np.zeros(n)
for rep in range(5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n):
        eng.forward_unit(x.shape[0], i, x, out)
        ev[i + 1].record()
    torch.cuda.synchronize()
    if rep:
        acc += [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
acc /= 4
print(os.environ.get("PCNN_TC_DEBUG", "0"), "total %.3f ms" % acc.sum(), " ".join("%.3f" % v for v in acc))
