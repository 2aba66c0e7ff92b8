# usage: VARS="A=1 A=2" CFGS="resnet20" bash tools/gpu_cmp_env.sh  -> ms_per_step per setting
mkdir -p gpurun_out
for v in base $VARS; do
  for c in ${CFGS:-resnet20}; do
    if [ $v = base ]; then python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/cmp_${c}_$v.json 2>gpurun_out/cmp_${c}_$v.err;
    else env $v python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/cmp_${c}_$v.json 2>gpurun_out/cmp_${c}_$v.err; fi
    echo "$v $c $(python -c "import json,sys;print(json.loads(open('gpurun_out/cmp_${c}_$v.json').read().strip().splitlines()[-1])['ms_per_step'])" 2>&1 | tail -1)"
  done
done
