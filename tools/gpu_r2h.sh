# timeline of every unit at the current build (A/B against the previous call's numbers), parity tests, then a stem trace
mkdir -p gpurun_out
for c in resnet18 vgg11 resnet20 resnet20_deg8; do python tools/time_all_units.py $c > gpurun_out/units_$c.txt 2>&1; done
grep -h total gpurun_out/units_*.txt | cut -c1-400
python -m pytest tests/test_gpu_configs.py tests/test_gpu_tc.py tests/test_gpu_units.py -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
if [ -n "$TRACE" ]; then
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
for u in $TRACE; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u resnet18 > gpurun_out/tr18_$u.txt 2>&1; tail -1 gpurun_out/tr18_$u.txt; done
fi
