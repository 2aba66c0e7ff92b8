mkdir -p gpurun_out
for rep in 1 2; do for v in 1 0; do
PCNN_SCRATCH_CB4=$v python bench.py --config resnet18 --steps 30 --warmup 5 --no-cpu --no-parity --no-redist-timing --secondary "" 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('cb4=$v', d['ms_per_step'], d['unit_ms'][:3])"
done; done
