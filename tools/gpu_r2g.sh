# CTA-0 pipeline traces of RN18 halo-tile layers (stage 1 N=64, stage 2 pair N=128, stage 3 pair)
mkdir -p gpurun_out
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
for u in 2 9 14; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u resnet18 > gpurun_out/tr18_$u.txt 2>&1; tail -1 gpurun_out/tr18_$u.txt; done
