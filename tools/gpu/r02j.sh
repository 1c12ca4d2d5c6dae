O=gpurun_out/r02j; mkdir -p $O
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_select_cluster" --launch-skip 10 --launch-count 1 -o $O/csel python bench.py --steps 3 --warmup 12 --no-cpu --no-e2e --island-load 8 > $O/ncu.log 2>&1
