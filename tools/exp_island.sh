#!/bin/bash
# time each experimental build in exp_libs/ at C4 on one GPU: the full island
# (P=65536) and one island's load at 4 and 8 GPUs (--island-load G)
for f in exp_libs/*.so; do
  for g in 0 4 8; do
    echo "== $f island-load $g"
    PGA_LIB=$f timeout 300 python bench.py --no-cpu --no-e2e --island-load $g 2>gpurun_out/exp_err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['population_per_gpu'], d['ms_per_step'], d['phase_ms_per_generation'])"
  done
done
