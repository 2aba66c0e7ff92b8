mkdir -p gpurun_out
for v in "2 1" "3 1" "3 2" "2 2"; do set -- $v
make -B -j16 NVEXTRA="-DPCNN_WAVE_MMA_WARPS=$1 -DPCNN_BLK_MMA_WARPS=$2" > /dev/null 2>&1
for rep in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "test_forward_matches_golden" 2>&1 | tail -1 | sed "s/^/wave=$1 blk=$2: /"; done
done
