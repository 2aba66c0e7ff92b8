mkdir -p gpurun_out
python -m pytest tests/test_gpu_tc.py -m gpu -q -k band > gpurun_out/t_band.txt 2>&1; tail -3 gpurun_out/t_band.txt
python bench.py --steps 20 --warmup 5 --config resnet18 --secondary vgg11 --no-cpu --no-redist-timing > gpurun_out/b18.json 2> gpurun_out/b18.err; tail -3 gpurun_out/b18.err
python -c "
import json;d=json.loads(open('gpurun_out/b18.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity']['max_rel_err'], d['unit_ms'][:6])
s=d['secondary']['vgg11'];print(s['ms_per_step'], s['roofline']['frac'], s['parity']['max_rel_err'], s['unit_ms'])
"
mkdir -p gpurun_out
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 1 resnet18 > gpurun_out/trb_resnet18_1.txt 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 1 vgg11 > gpurun_out/trb_vgg11_1.txt 2>&1
make -B -j16 > /dev/null 2>&1
