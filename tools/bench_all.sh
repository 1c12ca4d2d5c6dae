#!/bin/bash
# Every bench line of a round (run on a GPU box via gpurun): C1-C5, F1 plain and
# streamed, and the reference arm on C4; outputs gpurun_out/bench_<cfg>.json.
for c in C1 C2 C3; do
  timeout 600 python bench.py --config $c --steps 500 --warmup 5 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
done
timeout 600 python bench.py > gpurun_out/bench_C4.json 2>gpurun_out/bench_C4.err
timeout 900 python bench.py --config C5 --steps 500 --warmup 5 --no-cpu > gpurun_out/bench_C5.json 2>gpurun_out/bench_C5.err
timeout 600 python bench.py --config F1 --steps 3 --warmup 5 > gpurun_out/bench_F1.json 2>gpurun_out/bench_F1.err
timeout 600 python bench.py --config F1 --stream --steps 3 --warmup 5 > gpurun_out/bench_F1_stream.json 2>gpurun_out/bench_F1_stream.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_C4.json 2>gpurun_out/bench_ref_C4.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
for f in gpurun_out/bench_*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('ms_per_step'), d.get('value'), d.get('unit'))
except Exception as e: print('$f', 'FAILED', e)"; done
tail -1 gpurun_out/smoke.txt
