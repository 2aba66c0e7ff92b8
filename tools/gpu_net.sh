# whole-network kernel: probe, GPU tests, LeNet bench A/B
python tools/net_probe.py 2>&1 | tail -6
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/net_pytest.txt 2>&1; tail -3 gpurun_out/net_pytest.txt
for spec in "" "PCNN_NO_NET=1"; do
env $spec timeout 300 python bench.py --config lenet5 --steps 50 --warmup 5 --secondary "" --no-cpu --no-redist-timing 2>gpurun_out/net_bench_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(repr('$spec'), d['ms_per_step'], d['value'], d['e2e']['value'], d.get('parity',{}).get('max_rel_err'), d['gpu_launches'], d['roofline'].get('kernel'))"
done
