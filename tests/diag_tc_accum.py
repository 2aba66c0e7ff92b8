"""Diagnostic (not a test): error statistics of the tcgen05 3xTF32 path vs fp64."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
from helpers import chain
from oracle import levnet_oracle as O
from paper_2509_22857_b200.graph import ConvNode, InputNode, OutputNode
from paper_2509_22857_b200.runtime import Engine

rng = np.random.default_rng(0)
for cin, sign in ((64, 1), (512, 1), (2048, 1), (4608, 1), (512, 0), (4608, 0)):
    w = rng.uniform(0, 1, (64, cin, 1, 1)) / cin if sign else rng.normal(0, 1, (64, cin, 1, 1)) / np.sqrt(cin)
    g = chain([InputNode("in", cin, 4, 4), ConvNode("c", w, np.zeros(64), 1, 0), OutputNode("out")])
    x = rng.uniform(0, 1, (32, cin, 4, 4)) if sign else rng.normal(0, 1, (32, cin, 4, 4))
    want = np.stack([O.reference_eval(g, xi) for xi in x[:8]])
    for impl in (2, 1):
        got = Engine(g, impl=impl).forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()[:8]
        d = (got - want) / np.abs(want).max()
        print(f"cin={cin} positive={sign} impl={impl}: max|rel|={np.abs(d).max():.2e} mean={d.mean():.2e} std={d.std():.2e}")
