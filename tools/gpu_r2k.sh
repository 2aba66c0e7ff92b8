# A/B: scratch map of a pooled halo-tile conv in 4-channel blocks (scratch_cb4) vs the tensor's block width
mkdir -p gpurun_out
python tools/time_all_units.py resnet18 scratch_cb4=0 > gpurun_out/cb4_resnet18.txt 2>&1
grep -h total gpurun_out/cb4_resnet18.txt | cut -c1-120
python -m pytest tests/test_gpu_units.py tests/test_gpu_configs.py -m gpu -x -q -k "resnet18 or local or pool" > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
