timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
for c in C1 C2 C3; do
  timeout 600 python bench.py --config $c --steps 500 --warmup 5 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read()); print('$c', d['ms_per_step'], d['value'])"
done
