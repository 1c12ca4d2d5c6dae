# cluster-cache minimum cluster size 4 / 5 (default) / 6 at C4 and island-load 8
O=gpurun_out/r04b; mkdir -p $O
for r in 1 2; do
  for v in base cc4 cc6; do
    L=paper_1403_4099_b200/libpga.so; [ $v != base ] && L=paper_1403_4099_b200/libpga_$v.so
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
    PGA_LIB=$L timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_${v}_$r.json 2>> $O/bench.err
  done
done
