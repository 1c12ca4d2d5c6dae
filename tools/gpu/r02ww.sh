# breed parent-word loads: v3 (second parent unpredicated on the crossover draw), v4 (+ all chunks' words loaded first; libpga.so), prev (HEAD)
O=gpurun_out/r02ww; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "lockstep or breed or op_" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  for v in v4 v3 prev; do
    L=paper_1403_4099_b200/libpga.so; [ $v = v3 ] && L=paper_1403_4099_b200/libpga_v3.so; [ $v = prev ] && L=paper_1403_4099_b200/libpga_prev.so
    PGA_LIB=$L timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_${v}_$r.json 2>> $O/bench.err
    PGA_LIB=$L timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_${v}_$r.json 2>> $O/bench.err
  done
done
for v in v4 v3 prev; do
  L=paper_1403_4099_b200/libpga.so; [ $v = v3 ] && L=paper_1403_4099_b200/libpga_v3.so; [ $v = prev ] && L=paper_1403_4099_b200/libpga_prev.so
  PGA_LIB=$L timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_breed2 -c 12 --csv --log-file $O/breed_$v.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu_$v.log 2>&1
done
