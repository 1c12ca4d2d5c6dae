# rank selection up to P = 8192 only: selection tests + island loads
O=gpurun_out/r04a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_checks.py -q -x -k "cluster_select or ties or checks or invariants or identical" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do for g in 8 4 2; do timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_$r.json 2>> $O/bench.err; done; done
