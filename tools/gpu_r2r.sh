mkdir -p gpurun_out
for rep in 1 2; do
make -B -j16 > /dev/null 2>&1
for c in resnet20 resnet20_deg8; do python tools/time_all_units.py $c 2>&1 | grep total | cut -c1-150 | sed "s/^/base $c /"; done
make -B -j16 NVEXTRA=-DPCNN_SS_GROUPED > /dev/null 2>&1
for c in resnet20 resnet20_deg8; do python tools/time_all_units.py $c 2>&1 | grep total | cut -c1-150 | sed "s/^/grouped $c /"; done
done
