mkdir -p gpurun_out
python tools/plan_info.py resnet20 > gpurun_out/plan20.txt 2>&1
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
for u in 3 10 17 20; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u resnet20 > gpurun_out/tr_$u.txt 2>&1; done
