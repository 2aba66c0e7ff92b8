# A/B: epilogue warpgroup pairs on 64-channel halo tiles (epi_pairs 3) / every tile (4); precision table; e2e probe
mkdir -p gpurun_out
for c in resnet18 vgg11 resnet20; do
  python tools/time_all_units.py $c epi_pairs=3 epi_pairs=4 > gpurun_out/pairs_$c.txt 2>&1
done
python bench.py --steps 10 --warmup 3 --secondary "" --no-cpu > gpurun_out/prec_rn20.json 2> gpurun_out/prec_rn20.err
python tools/e2e_probe.py resnet20 > gpurun_out/e2e_probe.txt 2>&1
cat gpurun_out/pairs_*.txt | grep total
