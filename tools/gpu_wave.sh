timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/wave_pytest.txt 2>&1; tail -3 gpurun_out/wave_pytest.txt
python tools/plan_info.py resnet20 2>&1 | sed -n 1,12p
bash tools/gpu_opt_ab.sh resnet20 PCNN_BLOCKS=0
bash tools/gpu_opt_ab.sh resnet20_deg8
timeout 300 python bench.py --config resnet20 --steps 20 --warmup 5 --secondary "" --no-cpu --no-redist-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity'], [round(x*1e3,1) for x in d['unit_ms']])"
