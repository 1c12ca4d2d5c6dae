O=gpurun_out/f1probe; mkdir -p $O
timeout 600 python bench.py --config F1 --steps 3 --warmup 5 --no-cpu > $O/f1_a.json 2> $O/f1_a.err
timeout 600 python tools/f1_e2e_probe.py > $O/probe.txt 2>&1
timeout 600 python bench.py --config F1 --steps 3 --warmup 5 --no-cpu > $O/f1_b.json 2> $O/f1_b.err
