run() { (cd $1 && python bench.py --steps 30 --warmup 5 --no-cpu --no-redist-timing --no-parity --secondary "" 2>/dev/null || python bench.py --steps 30 --warmup 5 --no-cpu --no-redist-timing 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
for r in 1 2; do run old_r01; run .; done
