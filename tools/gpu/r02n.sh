O=gpurun_out/r02n; mkdir -p $O
for th in -1 0.1 0.25 1; do
  timeout 900 python bench.py --config C5 --fitness-only --steps 5 --warmup 3 --no-cpu --sparse-theta $th > $O/c5_fit_$th.json 2>> $O/bench.err
done
timeout 900 python bench.py --config C4 --fitness-only --steps 10 --warmup 3 --no-cpu > $O/c4_fit.json 2>> $O/bench.err
timeout 900 python bench.py --config C4 --fitness-only --steps 10 --warmup 3 --no-cpu --sparse-theta 1 > $O/c4_fit_1.json 2>> $O/bench.err
timeout 900 python bench.py --config C4 --fitness-only --steps 10 --warmup 3 --no-cpu --sparse-theta 0 > $O/c4_fit_0.json 2>> $O/bench.err
