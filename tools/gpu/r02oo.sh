# dynamic chromosome hand-out in the label-sparse pass (PGA_SP_STATIC=1 = per-block): parity + A/B
O=gpurun_out/r02oo; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cache.py tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_dyn_$r.json 2>> $O/bench.err
    PGA_SP_STATIC=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_static_$r.json 2>> $O/bench.err
  done
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_dyn_$r.json 2>> $O/bench.err
  PGA_SP_STATIC=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_static_$r.json 2>> $O/bench.err
done
