"""Per-instruction summary of an ncu --set full capture (source page, SASS):
total warp instructions, stall reasons, and the per-item path (instructions
executed a given number of times, e.g. once per epilogue chunk per warp).

  python tools/sass_items.py gpurun_out/x.ncu-rep [lo hi]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia, isamp, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
n = lambda r: int(r[ia] or 0)
print("warp instructions", sum(n(r) for r in data), "samples", sum(int(r[isamp] or 0) for r in data))
agg = {hdr[i]: sum(int(r[i] or 0) for r in data) for i in stall}
print("stalls", sorted(agg.items(), key=lambda kv: -kv[1])[:8])
hist = collections.Counter(n(r) for r in data if n(r))
print("exec-count classes (count x instrs):", sorted(hist.items(), key=lambda kv: -kv[0] * kv[1])[:8])
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    per = [r for r in data if lo <= n(r) <= hi]
    op = lambda r: r[src].split()[1] if r[src].strip().startswith("@") else r[src].split()[0]
    print(f"path [{lo},{hi}]: {len(per)} instrs, samples {sum(int(r[isamp] or 0) for r in per)}")
    print(collections.Counter(op(r) for r in per).most_common(30))
