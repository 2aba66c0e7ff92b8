make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=38 SS=1 ALL=1 python tools/trace_tc.py 2 resnet20 > gpurun_out/tr6_u2.txt 2>&1
PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=2086 SS=1 ALL=1 python tools/trace_tc.py 2 resnet20 > gpurun_out/tr6n_u2.txt 2>&1
make -B -j16 > /dev/null 2>&1
PCNN_TC_DEBUG=2048 python tools/time_unit_opts.py resnet20 2 debug=2048 debug=2054
