python -m pytest tests -m gpu -q > gpurun_out/t.txt 2>&1; tail -15 gpurun_out/t.txt
