"""Where the pipelined e2e time goes: repeated forward_host_many calls of n batches (RN20 by default)."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200 import _lib as _L
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
cfg = configs.CONFIGS[name]
g = bench.build_model(name)
eng, gr, _ = bench.redistributed_engine(g, cfg, _L.options_from_env())
b = cfg.batch
xh = torch.from_numpy(configs.make_input(cfg, batch=b, seed=2).astype(np.float32)).pin_memory()
x = xh.cuda()
out = torch.empty(eng.out_shape(b), dtype=torch.float32, device="cuda")
eng.forward(x, out)
stream = torch.cuda.current_stream()
def dev(n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        eng.forward(x, out, check=False)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
dev(5)
print("device, warm L2, back to back: %.4f ms/step" % dev(50))
staging = (torch.empty_like(x), torch.empty_like(x), torch.empty_like(out))
def pipe(n, sync=False):
    outs = [torch.empty(eng.out_shape(b), dtype=torch.float32).pin_memory() for _ in range(n)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    eng.forward_host_many([xh] * n, outs, staging=staging, sync=sync)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (t1 - t0) * 1e3
for n in (3, 3, 20, 20, 20, 100, 100):
    ms, cpu = pipe(n)
    print("n=%3d  %.3f ms total  %.4f ms/step  (cpu enqueue %.3f ms)" % (n, ms, ms / n, cpu))
