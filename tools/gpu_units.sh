mkdir -p gpurun_out
for c in resnet18 resnet20 vgg11; do
  python tools/plan_info.py $c > gpurun_out/pi_$c.txt 2>&1
  timeout 300 python tools/time_all_units.py $c debug=2 debug=4 debug=6 > gpurun_out/tu_$c.txt 2>&1
done
tail -n 5 gpurun_out/tu_*.txt
