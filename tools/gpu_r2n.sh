mkdir -p gpurun_out
python bench.py > gpurun_out/r02f_default_bench.json 2> gpurun_out/r02f_default_bench.err; tail -c 300 gpurun_out/r02f_default_bench.json
for c in vgg11 resnet18 lenet5 resnet20_deg8; do python bench.py --config $c --secondary "" > gpurun_out/r02f_${c}_bench.json 2> gpurun_out/r02f_${c}_bench.err; done
python -m pytest tests -m gpu -x -q > gpurun_out/r02f_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r02f_pytest_gpu.txt
python tools/time_all_units.py resnet18 > gpurun_out/units18.txt 2>&1; grep total gpurun_out/units18.txt | cut -c1-100
