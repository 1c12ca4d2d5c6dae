O=gpurun_out/r02v; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 0 1 0 1; do
  PGA_NO_MUTMASK=$v timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_nomm$v.json 2>> $O/bench.err
  PGA_NO_MUTMASK=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_nomm$v.json 2>> $O/bench.err
done
