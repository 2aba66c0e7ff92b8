mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_units.py -m gpu -x -q -k "resnet20" > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
for rep in 1 2 3; do for c in resnet20 resnet20_deg8; do timeout 300 python tools/time_all_units.py $c 2>&1 | grep total | cut -c1-110 | sed "s/^/$c /"; done; done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.txt 2>&1; tail -1 gpurun_out/t_all.txt
