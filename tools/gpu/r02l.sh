# A/B: cluster cache from n >= 4 vs n >= 5 (same box, alternating)
O=gpurun_out/r02l; mkdir -p $O
for r in 1 2; do
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/base_$r.json 2>> $O/bench.err
  PGA_LIB=exp_libs/libpga_cc4.so timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/cc4_$r.json 2>> $O/bench.err
done
PGA_LIB=exp_libs/libpga_cc4.so timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/cc4_1000.json 2>> $O/bench.err
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu --no-e2e > $O/base_1000.json 2>> $O/bench.err
