# whole-block dense CTAs in GA generations: full GPU suite + bench lines
O=gpurun_out/r02rr; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for g in 8 4 2; do
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}.json 2>> $O/bench.err
done
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4.json 2>> $O/bench.err
for c in C1 C2 C3; do timeout 300 python bench.py --config $c --steps 500 --warmup 5 --no-cpu --no-e2e > $O/$c.json 2>> $O/bench.err; done
