for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu --no-redist-timing --no-parity > gpurun_out/rep_$i.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/rep_$i.json').read().strip().splitlines()[-1])
s=d['secondary']['resnet18'];print('rn20', d['ms_per_step'], 'rn18', s['ms_per_step'], s['unit_ms'][6:10])
"
done
python bench.py --steps 20 --warmup 5 --config resnet18 --secondary resnet20 --no-cpu --no-redist-timing --no-parity > gpurun_out/rep_3.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/rep_3.json').read().strip().splitlines()[-1])
s=d['secondary']['resnet20'];print('rn18', d['ms_per_step'], d['unit_ms'][6:10], 'rn20', s['ms_per_step'])
"
