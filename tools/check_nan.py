"""Where do NaNs come from at benchmark batch size?"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200.runtime import Engine
from oracle import levnet_oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
cfg = configs.CONFIGS[name]
g = configs.build(name)
x = configs.make_input(cfg)
xt = torch.from_numpy(x.astype(np.float32)).cuda()
ref = O.eval_batch(g, x[:4])
for impl in (1, 2, 0):
    try:
        eng = Engine(g, impl=impl, options=_L.options_from_env())
    except Exception as e:
        print("impl", impl, "plan failed", e); continue
    for gr in (0, 1):
        y = eng.forward(xt, use_graph=bool(gr)).double().cpu().numpy()
        bad = np.argwhere(~np.isfinite(y))
        print(f"impl={impl} graph={gr} nonfinite={len(bad)} first={bad[:3].tolist()} err4={np.abs(y[:4]-ref).max()/np.abs(ref).max():.2e}")
