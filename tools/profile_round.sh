#!/bin/bash
# Run on a GPU box (via gpurun): plain bench lines (C4 default, F1 batched),
# ncu launch lists of the same commands, ncu --set full of the dominant
# kernels: k_fitness (dense sweep; label-sparse pass disabled so every block
# runs it) and k_breed2 for C4, k_fitness_sparse in the sparse regime (first
# generations), k_batch for F1.  Outputs in gpurun_out/.
set -e
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
DENSE="$CMD --sparse-theta 0"
F1="python bench.py --config F1 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1
$F1 > gpurun_out/prof_plain_f1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/prof_launches.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_batch --csv \
    --log-file gpurun_out/launches_f1.csv $F1 > gpurun_out/prof_launches_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fitness$|k_breed" -s 4 -c 2 \
    -o gpurun_out/prof_full $DENSE > gpurun_out/prof_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fitness_sparse -s 403 -c 1 \
    -o gpurun_out/prof_sparse python bench.py --steps 3 --warmup 410 --no-cpu --no-e2e \
    > gpurun_out/prof_sparse.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_batch -c 1 \
    -o gpurun_out/prof_f1 $F1 > gpurun_out/prof_f1.log 2>&1
echo profile-done
