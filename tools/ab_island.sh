for r in 1 2; do for f in exp_libs/a_head.so exp_libs/b_dup.so; do for g in 0 8; do
PGA_LIB=$f timeout 300 python bench.py --no-cpu --no-e2e --island-load $g 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['config']['population_per_gpu'], d['ms_per_step'], d['phase_ms_per_generation']['sparse_pass'])"
done; done; done
