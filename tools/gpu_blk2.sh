timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/blk_pytest.txt 2>&1; tail -2 gpurun_out/blk_pytest.txt
bash tools/gpu_opt_ab.sh resnet20 PCNN_BLOCKS=1
bash tools/gpu_opt_ab.sh resnet20_deg8
python tools/time_unit_opts.py resnet20 10 2>&1 | tail -1
python tools/time_unit_opts.py resnet20 17 2>&1 | tail -1
