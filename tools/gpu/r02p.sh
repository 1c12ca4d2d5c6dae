# k_fitness row tiles per CTA: A/B of F (dense pass and empty launches)
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for F in 1 2 4 8 0; do
  if [ $F = 0 ]; then unset PGA_FIT_F; else export PGA_FIT_F=$F; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > $O/c4_F$F.json 2>> $O/bench.err
  timeout 600 python bench.py --config C4 --fitness-only --steps 10 --warmup 3 --no-cpu --sparse-theta 0 > $O/c4fit_F$F.json 2>> $O/bench.err
done
unset PGA_FIT_F
timeout 900 python bench.py --config C5 --fitness-only --steps 5 --warmup 3 --no-cpu > $O/c5fit.json 2>> $O/bench.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8.json 2>> $O/bench.err
