mkdir -p gpurun_out
python -m pytest tests/test_gpu_tc.py -m gpu -q -k band > gpurun_out/t_band.txt 2>&1; tail -30 gpurun_out/t_band.txt
python -m pytest tests -m gpu -q > gpurun_out/t.txt 2>&1; tail -15 gpurun_out/t.txt
python bench.py --steps 20 --warmup 5 --config resnet18 --secondary vgg11 --no-cpu > gpurun_out/b18.json 2> gpurun_out/b18.err; tail -3 gpurun_out/b18.err
python -c "
import json;d=json.loads(open('gpurun_out/b18.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['families_ms_per_step'], d['parity']['max_rel_err'])
s=d['secondary']['vgg11'];print(s['ms_per_step'], s['roofline']['frac'], s['roofline']['families_ms_per_step'], s['parity']['max_rel_err'])
"
