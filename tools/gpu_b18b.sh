mkdir -p gpurun_out
python -m pytest tests/test_gpu_tc.py -m gpu -q -k band > gpurun_out/t_band.txt 2>&1; tail -3 gpurun_out/t_band.txt
python -m pytest tests/test_gpu_configs.py tests/test_gpu_units.py -m gpu -q -k "resnet18 or vgg" -x > gpurun_out/t18.txt 2>&1; tail -3 gpurun_out/t18.txt
