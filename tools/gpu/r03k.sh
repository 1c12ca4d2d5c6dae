# programmatic dependent launch on / off (PGA_PDL=0) with the round-2 final kernels
O=gpurun_out/r03k; mkdir -p $O
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_pdl_$r.json 2>> $O/bench.err
    PGA_PDL=0 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_nopdl_$r.json 2>> $O/bench.err
  done
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_pdl_$r.json 2>> $O/bench.err
  PGA_PDL=0 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_nopdl_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_pdl_$r.json 2>> $O/bench.err
  PGA_PDL=0 timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_nopdl_$r.json 2>> $O/bench.err
done
