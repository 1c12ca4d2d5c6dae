O=gpurun_out/r02y; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4.json 2>> $O/bench.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8.json 2>> $O/bench.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 4 > $O/il4.json 2>> $O/bench.err
timeout 600 python bench.py --config C3 --steps 300 --warmup 5 --no-cpu --no-e2e > $O/c3.json 2>> $O/bench.err
