# A/B of flag-synchronised launches (run under gpurun): tests first, bounded
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/t_flags.txt 2>&1; tail -2 gpurun_out/t_flags.txt
VARS="PCNN_FLAGS=0" CFGS="${CFGS:-resnet20 resnet18 resnet20_deg8}" timeout 600 bash tools/gpu_cmp_env.sh
