O=gpurun_out/r02x; mkdir -p $O
for r in 1 2; do timeout 600 python bench.py --config F1 --steps 3 --warmup 5 --no-cpu > $O/f1_$r.json 2>> $O/bench.err; done
timeout 600 python tools/f1_e2e_probe.py > $O/f1_probe.txt 2>&1
nproc > $O/nproc.txt; uptime >> $O/nproc.txt
