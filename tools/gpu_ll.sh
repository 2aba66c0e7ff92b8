mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
for c in vgg11 resnet18; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$c.csv python tools/fwd.py --config $c --iters 1 > /dev/null 2>&1
done
python - <<'PY'
import csv
for c in ["vgg11", "resnet18"]:
    rows = list(csv.reader(open(f"gpurun_out/ll_{c}.csv")))
    h = None
    out = []
    for r in rows:
        if r and r[0] == "ID": h = r; continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            out.append((d["Kernel Name"][:60], d["Grid Size"], float(d["Metric Value"]) / 1000))
    print(c)
    for k in out[-40:]: print("  %-60s %-12s %8.1f" % k)
PY
