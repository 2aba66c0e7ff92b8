mkdir -p gpurun_out
timeout 300 python tools/time_all_units.py resnet18 ss_pair=0 > gpurun_out/tp_resnet18.txt 2>&1
cat gpurun_out/tp_resnet18.txt | tail -8
timeout 300 python tools/time_all_units.py vgg11 ss_pair=0 > gpurun_out/tp_vgg11.txt 2>&1
cat gpurun_out/tp_vgg11.txt | tail -8
timeout 900 python -m pytest tests/test_gpu_units.py tests/test_gpu_configs.py -m gpu -x -q -k "resnet18 or vgg11" > gpurun_out/tp_tests.txt 2>&1
tail -15 gpurun_out/tp_tests.txt
