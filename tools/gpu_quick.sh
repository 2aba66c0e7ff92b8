mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
PCNN_TC_DEBUG=64 python tools/cta_times.py resnet20 > gpurun_out/ct20.txt 2>&1
PCNN_TC_DEBUG=64 python tools/cta_times.py resnet18 > gpurun_out/ct18.txt 2>&1
for c in resnet20 resnet18; do python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/b_$c.json 2>/dev/null; done
cat gpurun_out/b_*.json | python -c "import sys,json;[print(json.loads(l)['config']['workload'], json.loads(l)['ms_per_step'], json.loads(l)['e2e']['value']) for l in sys.stdin if l.startswith('{')]"
if [ -n "$TRACE_UNITS" ]; then make -B -j8 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1; for u in $TRACE_UNITS; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u resnet20 > gpurun_out/tr_$u.txt 2>&1; done; fi
