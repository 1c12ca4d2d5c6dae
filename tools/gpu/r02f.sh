# flakiness probe: the C5 full-size test repeated with PDL on and off
O=gpurun_out/r02f; mkdir -p $O
for pdl in 1 0; do for r in 1 2 3; do
  PGA_PDL=$pdl timeout 600 python -m pytest tests/test_gpu_paths.py -q -k "C5_fitness" > $O/c5_pdl${pdl}_$r.log 2>&1; echo "pdl=$pdl run=$r rc=$?" >> $O/summary.txt
done; done
PGA_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "C5" > $O/parity_c5.log 2>&1; echo "parity C5 rc=$?" >> $O/summary.txt
