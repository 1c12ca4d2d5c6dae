O=gpurun_out/r02o; mkdir -p $O
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 900 python tools/sanitize.py > $O/sanitize_check.log 2>&1; echo "rc=$?" >> $O/sanitize_check.log
timeout 900 python -m pytest tests/test_gpu_checks.py -q > $O/pytest_checks.log 2>&1; echo "rc=$?" >> $O/pytest_checks.log
