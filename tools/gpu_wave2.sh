timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/wave_pytest.txt 2>&1; tail -2 gpurun_out/wave_pytest.txt
bash tools/gpu_opt_ab.sh resnet20
bash tools/gpu_opt_ab.sh resnet20_deg8
python tools/time_unit_opts.py resnet20 2 2>&1 | tail -1
