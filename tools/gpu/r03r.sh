# q fused into the last merge level (P > 16384; PGA_NO_QFUSE=1 = k_qsum): lockstep + C4 A/B
O=gpurun_out/r03r; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_prev_$r.json 2>> $O/bench.err
done
