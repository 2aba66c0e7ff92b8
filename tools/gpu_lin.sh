timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/lin_pytest.txt 2>&1; tail -2 gpurun_out/lin_pytest.txt
for c in vgg11 resnet18 resnet20; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --secondary "" --no-cpu --no-redist-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['parity']['max_rel_err'], d['roofline']['families_ms_per_step'])"
done
