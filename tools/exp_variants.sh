#!/bin/bash
# time each experimental build in exp_libs/ with the default C4 bench
for f in exp_libs/*.so; do
  echo "== $f"
  PGA_LIB=$f timeout 300 python bench.py --no-cpu --no-e2e 2>gpurun_out/exp_err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms_per_generation'])"
done
