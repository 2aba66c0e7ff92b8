# A/B: conv_blk_kernel with one MMA warp per resident image (2) vs one warp (1); wave kernel at 3 warps
mkdir -p gpurun_out
for w in 1 2 1 2; do
make -B -j16 NVEXTRA="-DPCNN_BLK_MMA_WARPS=$w" > gpurun_out/mkb_$w.log 2>&1
for c in resnet20 resnet20_deg8; do timeout 300 python tools/time_all_units.py $c 2>&1 | grep total | cut -c1-110 | sed "s/^/blk_warps=$w $c /"; done
done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_units.py -m gpu -x -q -k "resnet20" > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
