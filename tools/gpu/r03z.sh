# with the borrow-chain compare and 512-item runs: rank selection vs sort path at island sizes; rank chunk 256 / 512 / 1024
O=gpurun_out/r03z; mkdir -p $O
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_base_$r.json 2>> $O/bench.err
    PGA_NO_RANKC=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_norankc_$r.json 2>> $O/bench.err
    for t in 256 1024; do
      PGA_LIB=paper_1403_4099_b200/libpga_rs$t.so timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_rs${t}_$r.json 2>> $O/bench.err
    done
  done
done
