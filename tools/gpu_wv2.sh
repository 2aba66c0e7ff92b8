mkdir -p gpurun_out
for c in resnet20 resnet20_deg8; do timeout 300 python tools/time_all_units.py $c > gpurun_out/wv2_$c.txt 2>&1; cat gpurun_out/wv2_$c.txt; done
timeout 900 python -m pytest tests -m gpu -x -q -k "resnet20 or image_resident or blocks or wave" > gpurun_out/wv2_tests.txt 2>&1; tail -3 gpurun_out/wv2_tests.txt
