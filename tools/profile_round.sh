#!/bin/bash
# Run on a GPU box (via gpurun): plain bench, ncu launch list of the same
# command, ncu --set full of the dominant kernel.  Outputs in gpurun_out/.
set -e
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/prof_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fitness|k_breed" -s 4 -c 2 \
    -o gpurun_out/prof_full $CMD > gpurun_out/prof_full.log 2>&1
echo profile-done
