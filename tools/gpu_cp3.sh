mkdir -p gpurun_out
for d in 0 2 4 6; do
PCNN_PAIR=4 PCNN_TC_DEBUG=$d PCNN_NO_GRAPH=1 PCNN_NO_PDL=1 timeout 120 python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/cp3_$d.txt 2>&1; echo "debug=$d: $(tail -1 gpurun_out/cp3_$d.txt)"
done
