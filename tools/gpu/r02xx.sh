# selection tie tests, pageable host state: e2e breakdown and C4 bench line
O=gpurun_out/r02xx; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "ties or cluster_select or free_running" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_breakdown.py 20 > $O/e2e_breakdown.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/c4.json 2>> $O/bench.err
