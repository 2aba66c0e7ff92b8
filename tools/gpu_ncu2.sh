mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/fwd.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:conv_ss -s 0 -c 1 -o gpurun_out/r02_rn18_stem python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/ncu1.log 2>&1
