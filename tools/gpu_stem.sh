mkdir -p gpurun_out
timeout 300 python tools/time_all_units.py resnet18 > gpurun_out/ts_resnet18.txt 2>&1
cat gpurun_out/ts_resnet18.txt
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/fwd18.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'conv_ss_kernel<16' -c 1 -o gpurun_out/stem18 python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/ncu_stem.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'localpool|ingest|conv_ss_kernel<16' --csv --log-file gpurun_out/stem_traffic.csv python tools/fwd.py --config resnet18 --iters 1 > /dev/null 2>&1
tail -3 gpurun_out/ncu_stem.log
