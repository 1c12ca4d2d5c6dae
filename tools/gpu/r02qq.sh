# empty dense launch at island loads: whole-block CTAs (PGA_FIT_F=64 -> nRT) vs default; C4 launch list with late masks
O=gpurun_out/r02qq; mkdir -p $O
for r in 1 2; do
  for g in 8 4; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_def_$r.json 2>> $O/bench.err
    PGA_FIT_F=64 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load $g > $O/il${g}_F_$r.json 2>> $O/bench.err
  done
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_C4.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_il8.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --island-load 8 > $O/ncu_il8.log 2>&1
