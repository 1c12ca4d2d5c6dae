O=gpurun_out/r02aa; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/c4_$r.json 2>> $O/bench.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_$r.json 2>> $O/bench.err
done
