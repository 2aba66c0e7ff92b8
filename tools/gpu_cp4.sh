mkdir -p gpurun_out
timeout 300 python tools/time_all_units.py resnet18 ss_pair=3 > gpurun_out/cp4_18.txt 2>&1; cat gpurun_out/cp4_18.txt
timeout 300 python tools/time_all_units.py vgg11 ss_pair=3 > gpurun_out/cp4_v.txt 2>&1; cat gpurun_out/cp4_v.txt
