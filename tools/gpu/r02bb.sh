O=gpurun_out/r02bb; mkdir -p $O
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_batch -c 1 -o $O/kbatch python bench.py --config F1 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu.log 2>&1
