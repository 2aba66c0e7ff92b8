mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bq_default.json 2> gpurun_out/bq_default.err
for c in vgg11 resnet20_deg8; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --secondary "" > gpurun_out/bq_$c.json 2>/dev/null; done
python - <<'PY'
import json
for f in ["bq_default", "bq_vgg11", "bq_resnet20_deg8"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, d["config"]["workload"], d["ms_per_step"], d["value"], d["roofline"]["frac"], d["parity"]["max_rel_err"], d["e2e"]["value"])
    for k, s in d.get("secondary", {}).items():
        print("  ", k, s["ms_per_step"], s["value"], s["roofline"]["frac"], s["parity"]["max_rel_err"], s["e2e"]["value"])
PY
timeout 300 python tools/time_all_units.py resnet18 debug=4 debug=6 > gpurun_out/tq_resnet18.txt 2>&1
cat gpurun_out/tq_resnet18.txt
tail -3 gpurun_out/bq_default.err
