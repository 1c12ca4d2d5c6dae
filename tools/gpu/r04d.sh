# cluster-cache slots per chromosome with CC_NMIN 4: 32 / 64 (default) / 128 (2^23 slots at C4)
O=gpurun_out/r04d; mkdir -p $O
for r in 1 2; do
  for per in 64 32 128; do
    PGA_CC_PER=$per timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${per}_$r.json 2>> $O/bench.err
    PGA_CC_PER=$per timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/c4long_${per}_$r.json 2>> $O/bench.err
  done
done
