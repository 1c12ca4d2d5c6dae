# non-migration generation as one graph (phase A deferred to pga_gen_breed; PGA_NO_FUSE_GEN=1 = two graphs)
O=gpurun_out/r03j; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_fuse_$r.json 2>> $O/bench.err
    PGA_NO_FUSE_GEN=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_split_$r.json 2>> $O/bench.err
  done
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_fuse_$r.json 2>> $O/bench.err
  PGA_NO_FUSE_GEN=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_split_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_fuse_$r.json 2>> $O/bench.err
  PGA_NO_FUSE_GEN=1 timeout 300 python bench.py --config C3 --steps 500 --warmup 5 --no-cpu --no-e2e > $O/c3_split_$r.json 2>> $O/bench.err
done
