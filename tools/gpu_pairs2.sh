for u in 1 8 15; do python tools/time_unit_opts.py resnet20 $u epi_pairs=1 2>&1 | tail -2; done
for u in 1 2 6; do python tools/time_unit_opts.py resnet18 $u epi_pairs=1 2>&1 | tail -2; done
for u in 1 3 5; do python tools/time_unit_opts.py vgg11 $u epi_pairs=1 2>&1 | tail -2; done
