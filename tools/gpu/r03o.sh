# ncu --set full of the island-scale kernels (one island of an 8-GPU C4 split)
O=gpurun_out/r03o; mkdir -p $O
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_fitness_sparse|k_breed2|k_rank_sel" --launch-skip 30 --launch-count 3 -o $O/il8 python bench.py --steps 3 --warmup 20 --no-cpu --no-e2e --island-load 8 > $O/ncu.log 2>&1
