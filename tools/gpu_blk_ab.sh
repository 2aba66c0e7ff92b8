# image-resident runs: parity tests, then A/B of image_blocks 0 / 1 / 2 on the RN20 step
timeout 300 python -m pytest tests/test_gpu_configs.py -q -m gpu -k image_resident -x 2>&1 | tail -3
bash tools/gpu_opt_ab.sh ${1:-resnet20} PCNN_BLOCKS=1 PCNN_BLOCKS=2
for b in 0 2; do
PCNN_BLOCKS=$b python bench.py --config ${1:-resnet20} --steps 20 --warmup 5 --no-cpu --no-redist-timing --secondary "" --no-parity 2>gpurun_out/blk_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['gpu_launches'], [round(x*1e3,1) for x in d['unit_ms']])"
done
