O=gpurun_out/r02q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_checks.py -q -x > $O/pytest_checks.log 2>&1; echo "rc=$?" >> $O/pytest_checks.log
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4.json 2>> $O/bench.err
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/c4_1000.json 2>> $O/bench.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8.json 2>> $O/bench.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > $O/c5_ga.json 2>> $O/bench.err
