#!/bin/bash
# Round profile evidence (run under gpurun from the repo root):
#   1. the bench (plain, must exit 0), then its kernel launch list under ncu
#      (gpu__time_duration per launch, cold-cache, serialised)
#   2. dram bytes of every tcgen05 conv launch of one forward (traffic)
#   3. one --set full capture of the largest conv launch (source-level stalls)
# Usage: tools/profile_round.sh <config> <round-tag> <full-capture kernel regex> <launch-skip>
set -e
# ncu's kernel replay fails on extended launches inside CUDA graphs: profile
# eager, plain launches (identical kernels; the launch list compares shares)
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
cfg=${1:-resnet20}; tag=${2:-r01}; kre=${3:-conv_ss_kernel}; skip=${4:-0}
mkdir -p gpurun_out
python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-redist-timing --no-parity --secondary "" > gpurun_out/${tag}_${cfg}_plain.json 2> gpurun_out/${tag}_${cfg}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'conv_|ingest|linear_kernel|eltwise|localpool|to_vector|copyout' \
    -c 600 --csv --log-file gpurun_out/${tag}_${cfg}_launches.csv \
    python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-redist-timing --no-parity --secondary "" > gpurun_out/${tag}_${cfg}_ncu_bench.log 2>&1
python tools/fwd.py --config $cfg --iters 1 > gpurun_out/${tag}_${cfg}_fwd.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:conv_ \
    --csv --log-file gpurun_out/${tag}_${cfg}_traffic.csv python tools/fwd.py --config $cfg --iters 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:$kre -s $skip -c 1 -o gpurun_out/${tag}_${cfg}_full \
    python tools/fwd.py --config $cfg --iters 1 > gpurun_out/${tag}_${cfg}_full.log 2>&1
echo profile done
