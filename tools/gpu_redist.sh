timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/rd_pytest.txt 2>&1; tail -2 gpurun_out/rd_pytest.txt
for c in resnet20 resnet18 vgg11; do python tools/time_redist.py $c 2>&1 | tail -1; done
python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
from paper_2509_22857_b200 import configs
for name in ("resnet20", "vgg11", "resnet18"):
    g = configs.build(name)
    print(name, json.dumps(bench.time_redistribution(g, configs.CONFIGS[name])))
PY
