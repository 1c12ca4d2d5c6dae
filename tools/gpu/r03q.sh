# merge levels with 32-bit positions (libpga_prev.so = 64-bit)
O=gpurun_out/r03q; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_checks.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_prev_$r.json 2>> $O/bench.err
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_merge" -c 9 --csv --log-file $O/m_new.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu.log 2>&1
PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_merge" -c 9 --csv --log-file $O/m_prev.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu2.log 2>&1
