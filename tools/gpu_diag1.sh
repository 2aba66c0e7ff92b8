# where do the stems and image-resident runs spend their time
python tools/plan_info.py resnet20 > gpurun_out/d1_plan20.txt 2>&1
python tools/plan_info.py resnet18 > gpurun_out/d1_plan18.txt 2>&1
python tools/time_unit_opts.py resnet18 1 debug=2 debug=4 debug=6 > gpurun_out/d1_rn18u1.txt 2>&1
python tools/time_unit_opts.py resnet18 2 debug=2 debug=4 debug=6 >> gpurun_out/d1_rn18u1.txt 2>&1
python tools/time_unit_opts.py resnet20 1 debug=2 debug=4 debug=6 > gpurun_out/d1_rn20.txt 2>&1
python tools/time_unit_opts.py resnet20 2 debug=2 debug=4 debug=6 >> gpurun_out/d1_rn20.txt 2>&1
python tools/time_unit_opts.py resnet20 10 image_blocks=1 image_blocks=0 >> gpurun_out/d1_rn20.txt 2>&1
python tools/time_unit_opts.py resnet20 17 image_blocks=1 >> gpurun_out/d1_rn20.txt 2>&1
cat gpurun_out/d1_*.txt
