# one-launch rank + SUS selection (k_rank_sel): parity + island-load A/B (PGA_NO_RANKC=1 = previous path)
O=gpurun_out/r02ll; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_replicated.py tests/test_gpu_checks.py -q -x -k "cluster_select or replicated or checks" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_rc_$r.json 2>> $O/bench.err
    PGA_NO_RANKC=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_old_$r.json 2>> $O/bench.err
  done
done
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_il8.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --island-load 8 > $O/ncu.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_il4.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --island-load 4 > $O/ncu4.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_rank_sel --launch-skip 5 --launch-count 1 -o $O/ranksel python bench.py --steps 3 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/ncu_full.log 2>&1
