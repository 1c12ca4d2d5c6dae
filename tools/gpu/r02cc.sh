O=gpurun_out/r02cc; mkdir -p $O
for th in -1 0.25 1; do
  timeout 600 python bench.py --config C3 --steps 300 --warmup 5 --no-cpu --no-e2e --sparse-theta $th > $O/c3_$th.json 2>> $O/bench.err
done
