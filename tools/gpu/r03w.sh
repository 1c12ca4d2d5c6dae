# run length 512 and merge sample spacing 32 / 128 (defaults 1024 / 64)
O=gpurun_out/r03w; mkdir -p $O
for v in r512 ms32 ms128; do
  PGA_LIB=paper_1403_4099_b200/libpga_$v.so timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "cluster_select or op_select" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
done
for r in 1 2 3; do
  for v in base r512 ms32 ms128; do
    L=paper_1403_4099_b200/libpga.so; [ $v != base ] && L=paper_1403_4099_b200/libpga_$v.so
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
  done
done
