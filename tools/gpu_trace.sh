# CTA-0 pipeline traces of halo-tile units (run under gpurun):  CFG=resnet18 UNITS="3 10" bash tools/gpu_trace.sh
mkdir -p gpurun_out
python tools/plan_info.py ${CFG:-resnet20} > gpurun_out/plan_${CFG:-resnet20}.txt 2>&1
make -B -j16 NVEXTRA=-DPCNN_SS_TRACE > /dev/null 2>&1
for u in $UNITS; do PCNN_NO_GRAPH=1 PCNN_TC_DEBUG=32 SS=1 ALL=1 python tools/trace_tc.py $u ${CFG:-resnet20} > gpurun_out/tr_${CFG:-resnet20}_$u.txt 2>&1; done
make -B -j16 > /dev/null 2>&1
