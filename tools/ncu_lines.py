"""Per-source-line summary of an ncu --set full --import-source capture:
instructions executed and warp-stall samples per CUDA line (the SASS rows
under each line summed), top N by stall samples.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [N] [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kre = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kre:
    cmd += ["-k", "regex:" + kre]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file, hdr = None, None
stats = {}
line_src = {}
total_s = total_i = 0
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (cur_file, int(r[0]))
        line_src[cur] = r[1].strip()
        continue
    try:
        samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        insts = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    s = stats.setdefault(cur, [0, 0, {}])
    s[0] += samples
    s[1] += insts
    op = re.sub(r"^\s*(@!?U?P\w+\s+)?", "", r[3]).split(" ")[0]
    s[2][op] = s[2].get(op, 0) + insts
    total_s += samples
    total_i += insts
print(f"total stall samples {total_s}, instructions executed {total_i}")
for key, (smp, ins, ops) in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    opstr = ",".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:4])
    print(f"{100 * smp / max(total_s, 1):5.1f}% {ins:9d}  {key[0]}:{key[1]:<5d} {line_src.get(key, '')[:70]:70s} {opstr}")
