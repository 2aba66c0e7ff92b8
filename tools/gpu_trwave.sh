make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 BLK=1 ALL=1 python tools/trace_tc.py 2 resnet20 > gpurun_out/trwave2.txt 2>&1
make -B -j16 > /dev/null 2>&1
tail -3 gpurun_out/trwave2.txt
