mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:'localpool' -c 1 --csv --log-file gpurun_out/pool_ncu.csv python tools/fwd.py --config resnet18 --iters 1 > /dev/null 2>&1
grep -E "localpool" gpurun_out/pool_ncu.csv | awk -F'","' '{print $5, $13, $14, $15}' | cut -c1-140
