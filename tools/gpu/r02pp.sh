# mutation masks beside statistics + selection for P > 8192 (PGA_NO_MUTMASK_LATE=1 = off): parity + C4 / il4 A/B
O=gpurun_out/r02pp; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_sparse.py tests/test_gpu_replicated.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_late_$r.json 2>> $O/bench.err
  PGA_NO_MUTMASK_LATE=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_off_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 2 > $O/il2_late_$r.json 2>> $O/bench.err
  PGA_NO_MUTMASK_LATE=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 2 > $O/il2_off_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 4 > $O/il4_late_$r.json 2>> $O/bench.err
  PGA_NO_MUTMASK_LATE=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 4 > $O/il4_off_$r.json 2>> $O/bench.err
done
