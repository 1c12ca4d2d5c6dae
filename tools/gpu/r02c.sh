# gpurun script: full GPU suite, then bench A/B (PDL on/off) at C4 and one island of an 8-GPU split
O=gpurun_out/r02c; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for pdl in 1 0 1; do
  PGA_PDL=$pdl timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/bench_pdl$pdl.json 2>> $O/bench.err
  PGA_PDL=$pdl timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_pdl$pdl.json 2>> $O/bench.err
done
