O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_replicated.py tests/test_gpu_graphs.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 900 python tools/sanitize.py > $O/sanitize.log 2>&1; echo "rc=$?" >> $O/sanitize.log
for r in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_$r.json 2>> $O/bench.err
PGA_NO_CSEL=1 timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8_nocsel_$r.json 2>> $O/bench.err
done
