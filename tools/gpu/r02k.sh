O=gpurun_out/r02k; mkdir -p $O
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_fitness_sparse|k_breed2" --launch-skip 20 --launch-count 2 -o $O/early python bench.py --steps 3 --warmup 12 --no-cpu --no-e2e > $O/ncu1.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_fitness_sparse|k_breed2" --launch-skip 800 --launch-count 2 -o $O/late python bench.py --steps 3 --warmup 410 --no-cpu --no-e2e > $O/ncu2.log 2>&1
