mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
for v in 1 0; do
PCNN_SCRATCH_CB4=$v ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum --clock-control none -k regex:'conv_ss_kernel|localpool' -c 2 --csv --log-file gpurun_out/cb4_ncu_$v.csv python tools/fwd.py --config resnet18 --iters 1 > /dev/null 2>&1
grep -E "conv_ss|localpool" gpurun_out/cb4_ncu_$v.csv | awk -F'","' '{print $5, $13, $15}' | cut -c1-60,90-200
done
