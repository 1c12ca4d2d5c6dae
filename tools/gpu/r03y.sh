# full GPU suite + device checks on the final build
O=gpurun_out/r03y; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 900 python tools/sanitize.py > $O/sanitize.log 2>&1; echo "rc=$?" >> $O/sanitize.log
