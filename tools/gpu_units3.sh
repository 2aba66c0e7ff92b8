mkdir -p gpurun_out
for c in resnet20 vgg11 resnet20_deg8; do
timeout 600 python tools/time_all_units.py $c ss_wide=0 pdl=0 > gpurun_out/tu3_$c.txt 2>&1
done
cat gpurun_out/tu3_*.txt
