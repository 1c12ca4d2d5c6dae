# with stream priorities: mutation masks beside the fitness pass at C4 (early) vs beside the selection (late, default)
O=gpurun_out/r03m; mkdir -p $O
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_late_$r.json 2>> $O/bench.err
  PGA_MUTMASK_FORCE=1 PGA_NO_MUTMASK_LATE=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_early_$r.json 2>> $O/bench.err
done
