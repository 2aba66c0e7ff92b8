# stem (RN18 unit 1) CTA-0 trace with four epilogue warpgroups (epi_pairs = 3) next to the default
mkdir -p gpurun_out
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 PCNN_PAIRS=3 python tools/trace_tc.py 1 resnet18 > gpurun_out/tr18_1_pairs3.txt 2>&1; tail -1 gpurun_out/tr18_1_pairs3.txt
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 PCNN_PAIRS=3 python tools/trace_tc.py 2 resnet18 > gpurun_out/tr18_2_pairs3.txt 2>&1; tail -1 gpurun_out/tr18_2_pairs3.txt
