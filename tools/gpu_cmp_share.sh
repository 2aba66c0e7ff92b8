mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
for sh in default 1 2 3; do
  if [ $sh = default ]; then unset PCNN_SS_SHARE; else export PCNN_SS_SHARE=$sh; fi
  for c in resnet20 resnet18; do python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/b_${c}_$sh.json 2>/dev/null; done
  echo "share=$sh $(cat gpurun_out/b_resnet20_$sh.json gpurun_out/b_resnet18_$sh.json | python -c "import sys,json;print([json.loads(l)['ms_per_step'] for l in sys.stdin if l.startswith('{')])")"
done
unset PCNN_SS_SHARE
PCNN_TC_DEBUG=64 python tools/cta_times.py resnet20 > gpurun_out/ct20.txt 2>&1
