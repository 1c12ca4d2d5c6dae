# C5 label-sparse pass: tests, C5 GA generations and fitness-only lines
O=gpurun_out/r02m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_paths.py -q -x > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > $O/c5_ga.json 2>> $O/bench.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e --sparse-theta 0 > $O/c5_ga_dense.json 2>> $O/bench.err
timeout 900 python bench.py --config C5 --fitness-only --steps 5 --warmup 3 > $O/c5_fit.json 2>> $O/bench.err
timeout 900 python bench.py --config C5 --fitness-only --steps 5 --warmup 3 --no-cpu --sparse-theta 0 > $O/c5_fit_dense.json 2>> $O/bench.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4.json 2>> $O/bench.err
