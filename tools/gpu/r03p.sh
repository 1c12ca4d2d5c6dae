# 96-bit borrow-chain key compare in the sorts / rank selection (libpga_prev.so = plain compares)
O=gpurun_out/r03p; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_checks.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for v in new prev; do
    L=paper_1403_4099_b200/libpga.so; [ $v = prev ] && L=paper_1403_4099_b200/libpga_prev.so
    PGA_LIB=$L timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_${v}_$r.json 2>> $O/bench.err
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
    PGA_LIB=$L timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_${v}_$r.json 2>> $O/bench.err
  done
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rank_sel|k_sort_runs|k_merge" -c 12 --csv --log-file $O/sel_new.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu.log 2>&1
PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rank_sel|k_sort_runs|k_merge" -c 12 --csv --log-file $O/sel_prev.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu2.log 2>&1
