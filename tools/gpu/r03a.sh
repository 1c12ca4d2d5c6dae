# parents per mate pair gathered once after selection (k_pairs; PGA_NO_PAIRS=1 = breed's sigma -> sel chain)
O=gpurun_out/r03a; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_sparse.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_pairs_$r.json 2>> $O/bench.err
  PGA_NO_PAIRS=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_old_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_pairs_$r.json 2>> $O/bench.err
  PGA_NO_PAIRS=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_old_$r.json 2>> $O/bench.err
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_breed2|k_pairs" -c 12 --csv --log-file $O/breed_pairs.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu.log 2>&1
