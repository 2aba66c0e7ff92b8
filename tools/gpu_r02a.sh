mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/b.json 2> gpurun_out/b.err; tail -3 gpurun_out/b.err
python -c "
import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['share_of_step'], d['parity'])
s=d['secondary']['resnet18'];print(s['ms_per_step'], s['roofline']['frac'], s['parity'])
"
