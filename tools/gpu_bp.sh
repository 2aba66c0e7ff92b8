mkdir -p gpurun_out
timeout 300 python tools/time_all_units.py vgg11 > gpurun_out/tb_vgg11.txt 2>&1; cat gpurun_out/tb_vgg11.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "vgg or bipool or bivar" > gpurun_out/tb_tests.txt 2>&1; tail -3 gpurun_out/tb_tests.txt
