# Timing A/B of a diagnostic build (run under gpurun): DIAG=-DPCNN_DIAG_NOPTAB CFGS="resnet20" bash tools/gpu_diag_build.sh
mkdir -p gpurun_out
for c in ${CFGS:-resnet20}; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-redist-timing > gpurun_out/diag_base_$c.json 2>/dev/null; done
make -B -j16 NVEXTRA="$DIAG" > /dev/null 2>&1
for c in ${CFGS:-resnet20}; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-redist-timing > gpurun_out/diag_$c.json 2>/dev/null; done
make -B -j16 > /dev/null 2>&1
for c in ${CFGS:-resnet20}; do echo "$c base $(python -c "import json;print(json.loads(open('gpurun_out/diag_base_$c.json').read().strip().splitlines()[-1])['ms_per_step'])") diag $(python -c "import json;print(json.loads(open('gpurun_out/diag_$c.json').read().strip().splitlines()[-1])['ms_per_step'])" 2>&1 | tail -1)"; done
