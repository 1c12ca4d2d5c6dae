# 32 cache slots per chromosome: full GPU suite + bench lines
O=gpurun_out/r04e; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $O/c4.json 2>> $O/bench.err
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/c4_1000.json 2>> $O/bench.err
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_100.json 2>> $O/bench.err
for g in 2 4 8; do timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il$g.json 2>> $O/bench.err; done
timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu > $O/c3.json 2>> $O/bench.err
timeout 900 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu > $O/c5ga.json 2>> $O/bench.err
