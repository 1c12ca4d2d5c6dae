# dense fold's Eq. 8 with the table-driven log: full GPU suite + dense A/B against libpga_prev.so
O=gpurun_out/r03d; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  timeout 600 python bench.py --config C4 --fitness-only --steps 20 --warmup 3 --no-cpu --no-e2e > $O/c4fit_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 600 python bench.py --config C4 --fitness-only --steps 20 --warmup 3 --no-cpu --no-e2e > $O/c4fit_prev_$r.json 2>> $O/bench.err
  timeout 900 python bench.py --config C5 --fitness-only --steps 6 --warmup 3 --no-cpu --no-e2e > $O/c5fit_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 900 python bench.py --config C5 --fitness-only --steps 6 --warmup 3 --no-cpu --no-e2e > $O/c5fit_prev_$r.json 2>> $O/bench.err
done
