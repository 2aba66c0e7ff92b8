mkdir -p gpurun_out
timeout 300 python tools/cmp_plans.py resnet18 PCNN_PAIR=2 > gpurun_out/cp_resnet18.txt 2>&1; cat gpurun_out/cp_resnet18.txt | head -30
timeout 300 python tools/time_all_units.py resnet18 ss_pair=2 > gpurun_out/cp_t18.txt 2>&1; cat gpurun_out/cp_t18.txt
timeout 300 python tools/time_all_units.py vgg11 ss_pair=2 > gpurun_out/cp_tv.txt 2>&1; cat gpurun_out/cp_tv.txt
