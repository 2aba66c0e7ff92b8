mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
python tools/timeline_gaps.py resnet20 2>&1 | tail -10
python tools/timeline_gaps.py resnet20_deg8 2>&1 | tail -10
