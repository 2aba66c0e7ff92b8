"""Timeline of the tcgen05 conv pipeline in CTA 0 (PCNN_TC_DEBUG |= 32; for the
halo-tile kernel (SS=1) build with `make -B NVEXTRA=-DPCNN_SS_TRACE` first)."""
import ctypes, os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs, _lib as L
from paper_2509_22857_b200 import _lib as _L
from paper_2509_22857_b200.runtime import Engine
unit = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = configs.build(sys.argv[2] if len(sys.argv) > 2 else "resnet20")
eng = Engine(g, options=_L.options_from_env())
cfgname = sys.argv[2] if len(sys.argv) > 2 else "resnet20"
x = torch.from_numpy(configs.make_input(configs.CONFIGS[cfgname]).astype(np.float32)).cuda()
out = eng.forward(x)
lib = L.lib()
fn = lib.pcnn_ss_trace if os.environ.get("SS") else lib.pcnn_tc_trace
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 65536)()
for i in range(unit):
    eng.forward_unit(x.shape[0], i, x, out)
torch.cuda.synchronize()
fn(buf, 65536)  # reset
eng.forward_unit(x.shape[0], unit, x, out)
torch.cuda.synchronize()
n = fn(buf, 65536)
ev = [(int(v) >> 48, int(v) & 0xFFFFFFFFFFFF) for v in buf[:n] if int(v)]
t0 = min(t for _, t in ev)
names = {13: "ep_acc", 14: "ep_math", 12: "cv_stfull", 11: "cv_aempty", 10: "mma_k4", 1: "cv_lds", 2: "cv_go", 3: "cv_done", 4: "mma_wait", 5: "mma_go", 6: "mma_done", 7: "ep_wait", 8: "ep_go", 9: "ep_done"}
if os.environ.get("BLK"):
    names = {1: "p_ext", 2: "p_w", 3: "m_accw", 4: "m_acc_ok", 5: "m_in_ok", 6: "m_w_ok", 7: "m_issued", 8: "e_wait", 9: "e_go", 10: "e_chunk"}
ev.sort(key=lambda e: e[1])
for tag, t in (ev if os.environ.get("ALL") else ev[:240]):
    print(f"{t - t0:8d} {names.get(tag >> 8, tag >> 8):9s} kb={tag & 0xff:02x}")
print("events", n, "span", max(t for _, t in ev) - t0)
