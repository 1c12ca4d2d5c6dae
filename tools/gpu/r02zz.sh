# graph IF node around the dense launch (PGA_NO_COND=1 = plain launch): tests + A/B
O=gpurun_out/r02zz; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_cond_$r.json 2>> $O/bench.err
  PGA_NO_COND=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_plain_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_cond_$r.json 2>> $O/bench.err
  PGA_NO_COND=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_plain_$r.json 2>> $O/bench.err
done
timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_cond.json 2>> $O/bench.err
PGA_NO_COND=1 timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_plain.json 2>> $O/bench.err
