# cluster-cache table size: 16 / 32 / 64 (default) slots per chromosome, C4 (2^20 / 2^21 / 2^22 slots)
O=gpurun_out/r03n; mkdir -p $O
for r in 1 2; do
  for per in 64 32 16; do
    PGA_CC_PER=$per timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${per}_$r.json 2>> $O/bench.err
    PGA_CC_PER=$per timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/c4long_${per}_$r.json 2>> $O/bench.err
  done
done
