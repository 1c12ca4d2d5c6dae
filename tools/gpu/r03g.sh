# k_rank_sel tile 512 (16 tiles at P = 8192, every SM busy) vs 1024
O=gpurun_out/r03g; mkdir -p $O
PGA_LIB=paper_1403_4099_b200/libpga_t512.so timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "cluster_select or ties" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_t1024_$r.json 2>> $O/bench.err
    PGA_LIB=paper_1403_4099_b200/libpga_t512.so timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_t512_$r.json 2>> $O/bench.err
  done
done
