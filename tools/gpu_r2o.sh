mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
python bench.py --config resnet18 --secondary "" --no-cpu --no-redist-timing 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['ms_per_step'], d['roofline']['frac'], d['parity']['max_rel_err']); [print(r) for r in d['unfused_stages']]"
