# CC_NMIN 4: full GPU suite + 1000-generation C4 A/B against 5 (libpga_prev.so)
O=gpurun_out/r04c; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/c4long_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/c4long_prev_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_prev_$r.json 2>> $O/bench.err
done
