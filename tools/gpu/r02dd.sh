O=gpurun_out/r02dd; mkdir -p $O
for c in C1 C2; do for th in -1 0.25; do
  timeout 600 python bench.py --config $c --steps 300 --warmup 5 --no-cpu --no-e2e --sparse-theta $th > $O/${c}_$th.json 2>> $O/bench.err
done; done
timeout 600 python bench.py --config C3 --steps 2000 --warmup 5 --no-cpu --no-e2e --sparse-theta 0.25 > $O/C3_long_0.25.json 2>> $O/bench.err
timeout 600 python bench.py --config C3 --steps 2000 --warmup 5 --no-cpu --no-e2e --sparse-theta 0 > $O/C3_long_0.json 2>> $O/bench.err
