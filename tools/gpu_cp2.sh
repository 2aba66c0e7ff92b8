mkdir -p gpurun_out
for v in 3 4; do
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/cmp_plans.py resnet18 PCNN_PAIR=$v > gpurun_out/cp2_$v.txt 2>&1; tail -8 gpurun_out/cp2_$v.txt
done
