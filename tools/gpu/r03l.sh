# stream priorities: main stream high, side stream low (PGA_NO_PRIO=1 = default priorities)
O=gpurun_out/r03l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_paths.py -q -x -k "graph or lockstep" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_prio_$r.json 2>> $O/bench.err
    PGA_NO_PRIO=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_noprio_$r.json 2>> $O/bench.err
  done
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_prio_$r.json 2>> $O/bench.err
  PGA_NO_PRIO=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_noprio_$r.json 2>> $O/bench.err
done
