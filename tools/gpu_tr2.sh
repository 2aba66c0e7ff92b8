mkdir -p gpurun_out
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 1 resnet18 > gpurun_out/trb_resnet18_1.txt 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py 1 vgg11 > gpurun_out/trb_vgg11_1.txt 2>&1
make -B -j16 > /dev/null 2>&1
