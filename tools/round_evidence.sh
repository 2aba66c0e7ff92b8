#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   tests, smoke, the default bench line, every config's bench line, the
#   reference arm, then tools/profile_round.sh for the two headline configs.
# Usage: tools/round_evidence.sh <round-tag>
tag=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.txt 2>&1; tail -1 gpurun_out/${tag}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.txt 2>&1; tail -1 gpurun_out/${tag}_smoke.txt
python bench.py > gpurun_out/${tag}_default_bench.json 2> gpurun_out/${tag}_default_bench.err; tail -c 400 gpurun_out/${tag}_default_bench.json
python bench.py --impl reference > gpurun_out/${tag}_reference_bench.json 2> gpurun_out/${tag}_reference_bench.err
for c in lenet5 resnet20_deg8 vgg11 resnet18; do
  python bench.py --config $c --secondary "" > gpurun_out/${tag}_${c}_bench.json 2> gpurun_out/${tag}_${c}_bench.err
done
bash tools/profile_round.sh resnet20 $tag conv_wave 0 > gpurun_out/${tag}_prof20.log 2>&1; tail -1 gpurun_out/${tag}_prof20.log
bash tools/profile_round.sh resnet18 $tag conv_ss 14 > gpurun_out/${tag}_prof18.log 2>&1; tail -1 gpurun_out/${tag}_prof18.log
