timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pairs_pytest.txt 2>&1; tail -3 gpurun_out/pairs_pytest.txt
bash tools/gpu_opt_ab.sh resnet18 PCNN_PAIRS=1
bash tools/gpu_opt_ab.sh resnet20 PCNN_PAIRS=1
bash tools/gpu_opt_ab.sh vgg11 PCNN_PAIRS=1
timeout 300 python bench.py --config resnet18 --steps 20 --warmup 5 --secondary "" --no-cpu --no-redist-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity']['max_rel_err'], [round(x*1e3,1) for x in d['unit_ms']])"
