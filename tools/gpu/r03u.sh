# sparse pass: Zobrist keys + fixed-point diagonal staged in shared memory (libpga_prev.so = L2 loads)
O=gpurun_out/r03u; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  for v in new prev; do
    L=paper_1403_4099_b200/libpga.so; [ $v = prev ] && L=paper_1403_4099_b200/libpga_prev.so
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
    PGA_LIB=$L timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_${v}_$r.json 2>> $O/bench.err
  done
done
