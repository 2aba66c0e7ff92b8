# A/B: concat-mode MMAs grouped by shape (all N = 2NT, then all N = NT) vs interleaved per tap
mkdir -p gpurun_out
python tools/time_all_units.py resnet18 > gpurun_out/grp_base.txt 2>&1
make -B -j16 NVEXTRA=-DPCNN_SS_GROUPED > /dev/null 2>&1
python tools/time_all_units.py resnet18 > gpurun_out/grp_on.txt 2>&1
python tools/time_all_units.py resnet20 >> gpurun_out/grp_on.txt 2>&1
python tools/time_all_units.py vgg11 >> gpurun_out/grp_on.txt 2>&1
grep -h total gpurun_out/grp_base.txt gpurun_out/grp_on.txt | cut -c1-160
python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "redistributed_forward" > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
