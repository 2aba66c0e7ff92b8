# A/B of plan options on the bench step time: bash tools/gpu_opt_ab.sh resnet20 "PCNN_X=1" ...
cfg=$1; shift
for spec in "" "$@"; do
  for rep in 1 2; do
    env $spec python bench.py --config $cfg --steps 30 --warmup 5 --secondary "" --no-cpu --no-redist-timing --no-parity 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', repr('$spec'), d['ms_per_step'], d['e2e']['value'])"
  done
done
