# gpurun script: cluster selection -- new lockstep tests, GPU suite, benches (cluster on/off)
O=gpurun_out/r02g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "cluster_select or C5 or foreign" > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 0 1 0; do
  PGA_NO_CSEL=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_nocsel$v.json 2>> $O/bench.err
  PGA_NO_CSEL=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 4 > $O/il4_nocsel$v.json 2>> $O/bench.err
done
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/bench.json 2>> $O/bench.err
