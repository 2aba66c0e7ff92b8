mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/fwd18.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_ss -c 1 -o gpurun_out/stem18 python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/ncu_stem.log 2>&1
tail -2 gpurun_out/ncu_stem.log
