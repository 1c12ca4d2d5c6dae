O=gpurun_out/r02t; mkdir -p $O
timeout 600 python tools/f1_e2e_probe.py > $O/f1_probe.txt 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"k_fitness\b|k_fitness\(" --launch-skip 8 --launch-count 1 -o $O/c4_dense python bench.py --steps 3 --warmup 5 --no-cpu --no-e2e --sparse-theta 0 > $O/ncu_dense.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > $O/c4.json 2>> $O/bench.err
