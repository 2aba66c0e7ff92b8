mkdir -p gpurun_out
export PCNN_PAIR=4 PCNN_NO_PDL=1 PCNN_NO_GRAPH=1
timeout 900 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python tools/fwd.py --config resnet18 --iters 1 > gpurun_out/san.txt 2>&1
head -60 gpurun_out/san.txt
