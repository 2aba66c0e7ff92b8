# A/B: bash tools/gpu_ab.sh <dirA> <dirB> [config] -- two builds on the same box, alternating
cfg=${3:-resnet20}
run() { (cd $1 && python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu --no-redist-timing --no-parity --secondary "" 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', '$cfg', d['ms_per_step'], [round(x*1e3,1) for x in d.get('unit_ms', [])])"; }
for r in 1 2; do run $1; run $2; done
