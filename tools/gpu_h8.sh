mkdir -p gpurun_out
for c in resnet20 resnet20_deg8; do timeout 300 python tools/time_all_units.py $c > gpurun_out/th_$c.txt 2>&1; cat gpurun_out/th_$c.txt; done
