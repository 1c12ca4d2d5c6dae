# breed prefetch variants on one box: v1 (mask words before the plan; libpga.so), v2 (+ stop flag / generation / mate slots; libpga_v2.so), prev (HEAD)
O=gpurun_out/r02uu; mkdir -p $O
for r in 1 2 3; do
  for v in v1 v2 prev; do
    L=paper_1403_4099_b200/libpga.so; [ $v = v2 ] && L=paper_1403_4099_b200/libpga_v2.so; [ $v = prev ] && L=paper_1403_4099_b200/libpga_prev.so
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
  done
done
for v in v1 v2 prev; do
  L=paper_1403_4099_b200/libpga.so; [ $v = v2 ] && L=paper_1403_4099_b200/libpga_v2.so; [ $v = prev ] && L=paper_1403_4099_b200/libpga_prev.so
  PGA_LIB=$L timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_breed2 -c 12 --csv --log-file $O/breed_$v.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu_$v.log 2>&1
done
