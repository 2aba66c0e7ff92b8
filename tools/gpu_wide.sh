# producer lanes A/B: unit times (RN18 units 1,2,8,13; RN20 units 2, 8) and the steps
python tools/time_unit_opts.py resnet18 2 ss_wide=0 debug=6 ss_wide=0,debug=6 2>&1 | tail -4
python tools/time_unit_opts.py resnet18 8 ss_wide=0 2>&1 | tail -2
python tools/time_unit_opts.py resnet18 13 ss_wide=0 2>&1 | tail -2
python tools/time_unit_opts.py resnet18 1 ss_wide=0 2>&1 | tail -2
python tools/time_unit_opts.py resnet20 2 ss_wide=0 2>&1 | tail -2
python tools/time_unit_opts.py resnet20 8 ss_wide=0 2>&1 | tail -2
bash tools/gpu_opt_ab.sh resnet18 PCNN_WIDE=0
bash tools/gpu_opt_ab.sh resnet20 PCNN_WIDE=0
bash tools/gpu_opt_ab.sh vgg11 PCNN_WIDE=0
