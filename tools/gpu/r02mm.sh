# k_rank_sel chunk size A/B (RS_T 256 / 512 / 1024) at island loads 8 and 4
O=gpurun_out/r02mm; mkdir -p $O
for r in 1 2; do
  for g in 8 4; do
    for v in rs256 rs1024; do
      PGA_LIB=paper_1403_4099_b200/libpga_$v.so timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_${v}_$r.json 2>> $O/bench.err
    done
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_rs512_$r.json 2>> $O/bench.err
  done
done
PGA_LIB=paper_1403_4099_b200/libpga_rs256.so timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "cluster_select" > $O/pytest256.log 2>&1; echo "rc=$?" >> $O/pytest256.log
