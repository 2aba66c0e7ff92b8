# ncu --set full of the RN18 stem launch (conv_ss_kernel<16,..>, first conv_ss launch of one forward)
mkdir -p gpurun_out
export PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
ncu --set full --import-source on --clock-control none -k regex:conv_ss_kernel -s 0 -c 1 -o gpurun_out/stem18_full -f \
    python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/stem18_full.log 2>&1
tail -2 gpurun_out/stem18_full.log
