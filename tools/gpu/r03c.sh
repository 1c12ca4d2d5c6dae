# 8-way merge levels (PGA_NO_MERGE8=1 = 4-way): selection parity + C4 A/B + launch list
O=gpurun_out/r03c; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_replicated.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_m8_$r.json 2>> $O/bench.err
  PGA_NO_MERGE8=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_m4_$r.json 2>> $O/bench.err
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_merge|k_sort_runs" -c 12 --csv --log-file $O/merge8.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu.log 2>&1
