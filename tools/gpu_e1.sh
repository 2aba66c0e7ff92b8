mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
for c in resnet20 resnet20_deg8; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-redist-timing --secondary "" > gpurun_out/e1_$c.json 2>gpurun_out/e1_$c.err
  PCNN_BLOCKS=0 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-redist-timing --secondary "" > gpurun_out/e1_${c}_noblk.json 2>gpurun_out/e1_${c}_noblk.err
done
cat gpurun_out/e1_*.json | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'], d['ms_per_step'], d['gpu_launches'], d.get('parity',{}).get('max_rel_err'), [u for u in d['unit_ms'] if u])"
