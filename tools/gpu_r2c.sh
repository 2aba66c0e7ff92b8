mkdir -p gpurun_out
for c in resnet20 resnet18 vgg11 lenet5 resnet20_deg8; do
timeout 300 python tools/time_all_units.py $c pdl=0 > gpurun_out/tc_$c.txt 2>&1
done
tail -n 4 gpurun_out/tc_*.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tc_tests.txt 2>&1
tail -15 gpurun_out/tc_tests.txt
