python -m pytest tests/test_gpu_tc.py -q -m gpu -k band 2>&1 | tail -1
for c in resnet18 vgg11 resnet20; do
python bench.py --steps 20 --warmup 5 --config $c --secondary "" --no-cpu --no-redist-timing --no-parity > gpurun_out/bb_$c.json 2>/dev/null
PCNN_NO_BAND=1 python bench.py --steps 20 --warmup 5 --config $c --secondary "" --no-cpu --no-redist-timing --no-parity > gpurun_out/bn_$c.json 2>/dev/null
python -c "
import json
for f in ['gpurun_out/bb_$c.json','gpurun_out/bn_$c.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print('$c', f[11:13], d['ms_per_step'], d['unit_ms'][:8])
"
done
