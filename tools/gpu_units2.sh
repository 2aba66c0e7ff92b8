mkdir -p gpurun_out
timeout 600 python tools/time_all_units.py resnet18 ss_mt=2 ss_mt=2,debug=6 ss_mt=2,streamk_fill=0.9 streamk_fill=0.9 streamk=0 ss_wide=0 > gpurun_out/tu2_resnet18.txt 2>&1
cat gpurun_out/tu2_resnet18.txt
