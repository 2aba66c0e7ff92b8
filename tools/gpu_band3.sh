python tools/plan_info.py vgg11 2>&1 | head -20
for u in 1 3 5 7 9; do python tools/time_unit_opts.py vgg11 $u band_pool=1 2>&1 | tail -2; done
python tools/time_unit_opts.py resnet18 1 band_pool=1 2>&1 | tail -2
timeout 300 python bench.py --config vgg11 --steps 20 --warmup 5 --secondary "" --no-cpu --no-redist-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['families_ms_per_step'], [round(x*1e3,1) for x in d['unit_ms']])"
PCNN_BAND=1 timeout 300 python bench.py --config vgg11 --steps 20 --warmup 5 --secondary "" --no-cpu --no-redist-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['families_ms_per_step'], [round(x*1e3,1) for x in d['unit_ms']])"
