"""Run a few redistributed forwards of one config (profiling driver for ncu)."""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200.runtime import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="resnet20")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--impl", type=int, default=0)
ap.add_argument("--graph", type=int, default=0)
args = ap.parse_args()
cfg = configs.CONFIGS[args.config]
g = configs.build(args.config)
eng = Engine(g, impl=args.impl, options=_L.options_from_env())
x = torch.from_numpy(configs.make_input(cfg).astype(np.float32)).cuda()
for _ in range(args.iters):
    y = eng.forward(x, use_graph=bool(args.graph))
torch.cuda.synchronize()
print("ok", float(y.abs().mean()))
