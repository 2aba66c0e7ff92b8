# A/B: MMA-issuing warps of conv_wave_kernel (2 vs 3 vs 4)
mkdir -p gpurun_out
for w in 2 3 4 2 3; do
make -B -j16 NVEXTRA="-DPCNN_WAVE_MMA_WARPS=$w" > gpurun_out/mk_$w.log 2>&1
for c in resnet20 resnet20_deg8; do timeout 300 python tools/time_all_units.py $c 2>&1 | grep total | cut -c1-110 | sed "s/^/warps=$w $c /"; done
done
make -B -j16 NVEXTRA="-DPCNN_WAVE_MMA_WARPS=3" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "resnet20" > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
grep -h "conv_wave_kernel" gpurun_out/mk_3.log gpurun_out/mk_4.log | grep -i spill | cut -c1-200
