mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
python tools/plan_info.py resnet18 > gpurun_out/plan_resnet18.txt 2>&1
python tools/plan_info.py resnet20 > gpurun_out/plan_resnet20.txt 2>&1
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
for u in 1 2 3 10; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u resnet20 > gpurun_out/tr_resnet20_$u.txt 2>&1; done
for u in 1 3; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u resnet18 > gpurun_out/tr_resnet18_$u.txt 2>&1; done
make -B -j16 > /dev/null 2>&1
