mkdir -p gpurun_out
timeout 300 python tools/time_all_units.py resnet18 debug=2048 debug=6 debug=2054 ss_pair=0,debug=6 ss_pair=0,debug=2054 > gpurun_out/tw_resnet18.txt 2>&1
cat gpurun_out/tw_resnet18.txt
