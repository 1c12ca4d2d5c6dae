# Round-2 bench lines and captures -> gpurun_out/final/
O=gpurun_out/final10; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
for c in C1 C2 C3; do
  timeout 600 python bench.py --config $c --steps 500 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --steps 1000 --warmup 5 --no-cpu > $O/bench_C4_1000.json 2> $O/bench_C4_1000.err
timeout 900 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu > $O/bench_C5_ga.json 2> $O/bench_C5_ga.err
timeout 900 python bench.py --config C5 --fitness-only --steps 10 --warmup 3 > $O/bench_C5_fit.json 2> $O/bench_C5_fit.err
timeout 900 python bench.py --config C4 --fitness-only --steps 20 --warmup 3 > $O/bench_C4_fit.json 2> $O/bench_C4_fit.err
for g in 2 4 8; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/island_load_$g.json 2> $O/island_load_$g.err
done
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --mode replicated > $O/bench_C4_replicated.json 2> $O/bench_C4_rep.err
timeout 600 python bench.py --config F1 --steps 3 --warmup 5 > $O/bench_F1.json 2> $O/bench_F1.err
timeout 600 python bench.py --config F1 --stream --steps 3 --warmup 5 > $O/bench_F1_stream.json 2> $O/bench_F1_stream.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_C4.json 2> $O/bench_ref_C4.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_C4.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_fitness_sparse|k_breed2" --launch-skip 20 --launch-count 2 -o $O/c4_window python bench.py --steps 3 --warmup 12 --no-cpu --no-e2e > $O/ncu_full.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"k_fitness\b|k_fitness\(" --launch-skip 8 --launch-count 1 -o $O/c4_dense python bench.py --steps 3 --warmup 5 --no-cpu --no-e2e --sparse-theta 0 > $O/ncu_dense.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_il8.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --island-load 8 > $O/ncu_il8.log 2>&1
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
