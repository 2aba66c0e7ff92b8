cd old_r01 && PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 21 resnet20 > ../gpurun_out/tr21_old.txt 2>&1; cd ..
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 21 resnet20 > gpurun_out/tr21_new.txt 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 20 resnet20 > gpurun_out/tr20_new.txt 2>&1
make -B -j16 > /dev/null 2>&1
