# library memory pool for context buffers: full GPU suite, e2e breakdown, C4 bench line (e2e)
O=gpurun_out/r03f; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_breakdown.py 20 > $O/e2e_breakdown.txt 2>&1
for r in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/c4_$r.json 2>> $O/bench.err; done
timeout 600 python bench.py --config F1 --steps 3 --warmup 5 --no-cpu > $O/f1.json 2>> $O/bench.err
timeout 600 python bench.py --config F1 --stream --steps 3 --warmup 5 --no-cpu > $O/f1s.json 2>> $O/bench.err
