# merge-level CTA size: 128 / 256 (default) / 512 threads
O=gpurun_out/r03v; mkdir -p $O
for t in 512 128; do
  PGA_LIB=paper_1403_4099_b200/libpga_m$t.so timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "cluster_select or op_select" > $O/pytest_$t.log 2>&1; echo "rc=$?" >> $O/pytest_$t.log
done
for r in 1 2 3; do
  for t in 256 512 128; do
    L=paper_1403_4099_b200/libpga.so; [ $t != 256 ] && L=paper_1403_4099_b200/libpga_m$t.so
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${t}_$r.json 2>> $O/bench.err
  done
done
