O=gpurun_out/r02u; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py tests/test_gpu_paths.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --config C4 --fitness-only --steps 20 --warmup 3 --no-cpu --sparse-theta 0 > $O/c4_fit.json 2>> $O/bench.err
timeout 900 python bench.py --config C5 --fitness-only --steps 10 --warmup 3 --no-cpu > $O/c5_fit.json 2>> $O/bench.err
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > $O/c4.json 2>> $O/bench.err
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"k_fitness\b|k_fitness\(" --launch-skip 8 --launch-count 1 -o $O/c4_dense python bench.py --steps 3 --warmup 5 --no-cpu --no-e2e --sparse-theta 0 > $O/ncu_dense.log 2>&1
