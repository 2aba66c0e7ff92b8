mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
python tools/fwd.py --config resnet20 --iters 1 > gpurun_out/fwd20.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_wave -c 1 -o gpurun_out/wave20 python tools/fwd.py --config resnet20 --iters 1 > gpurun_out/ncu_wave.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_blk -c 1 -o gpurun_out/blk20 python tools/fwd.py --config resnet20 --iters 1 > gpurun_out/ncu_blk.log 2>&1
tail -1 gpurun_out/ncu_wave.log gpurun_out/ncu_blk.log
