O=gpurun_out/r02i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "cluster_select or replicated or islands" > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 0 1; do
  PGA_NO_CSEL=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_nocsel$v.json 2>> $O/bench.err
done
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 4 > $O/il4.json 2>> $O/bench.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/bench.json 2>> $O/bench.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_il8.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --island-load 8 > $O/ncu2.log 2>&1
