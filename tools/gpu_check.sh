#!/bin/bash
# One gpurun pass: GPU tests, compute-sanitizer over tools/sanitize.py, bench.
# usage: tools/gpu_check.sh TAG [pytest-args...]
TAG=${1:-r02}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 "$@" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
if [ -z "$NO_SAN" ]; then
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py > $OUT/sanitize_$t.log 2>&1
  echo "rc=$?" >> $OUT/sanitize_$t.log
done
fi
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
