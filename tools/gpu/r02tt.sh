# breed: stop flag, generation, mate slots and mask words in the first round trip (A/B against libpga_prev.so)
O=gpurun_out/r02tt; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_prev_$r.json 2>> $O/bench.err
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_new_$r.json 2>> $O/bench.err
  PGA_LIB=paper_1403_4099_b200/libpga_prev.so timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_prev_$r.json 2>> $O/bench.err
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_breed2 -c 12 --csv --log-file $O/breed_new.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e > $O/ncu.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_breed2 -c 12 --csv --log-file $O/breed_il8.csv python bench.py --steps 3 --warmup 8 --no-cpu --no-e2e --island-load 8 > $O/ncu2.log 2>&1
