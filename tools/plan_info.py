"""Print per-unit implementation and tensor formats of a config's plan."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200.runtime import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
cfg = configs.CONFIGS[name]
eng = Engine(configs.build(name), options=_L.options_from_env())
p = eng.plan(cfg.batch)
names = {1: "ingest", 2: "conv", 3: "linear", 8: "localpool", 10: "globalpool", 11: "flatten", 12: "copyout"}
for i, u in enumerate(eng.lw.units):
    k = u["kind"]
    s = f"{i:2d} {names.get(k, k):9s} impl={p.unit_impl(i)}"
    if k == 2:
        s += f" {u['cin']}->{u['cout']} k{u['kh']} s{u['stride']} in_fmt={p.tensor_split(u['in_'])} out_fmt={p.tensor_split(u['out'])}"
    print(s)
