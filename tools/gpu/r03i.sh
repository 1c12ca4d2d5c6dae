# occupancy knobs at island sizes: breed 3 CTAs/SM (libpga_b3.so), sparse pass 3 CTAs/SM (libpga_sp3.so)
O=gpurun_out/r03i; mkdir -p $O
for r in 1 2; do
  for v in base b3 sp3; do
    L=paper_1403_4099_b200/libpga.so; [ $v = b3 ] && L=paper_1403_4099_b200/libpga_b3.so; [ $v = sp3 ] && L=paper_1403_4099_b200/libpga_sp3.so
    for g in 8 4; do
      PGA_LIB=$L timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_${v}_$r.json 2>> $O/bench.err
    done
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
  done
done
