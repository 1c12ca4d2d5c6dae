# the whole GPU suite under the device-check build (invariant counters must stay 0)
O=gpurun_out/r03b; mkdir -p $O
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 2400 python -m pytest tests/ -q -x -m gpu -s > $O/pytest_checks.log 2>&1; echo "rc=$?" >> $O/pytest_checks.log
