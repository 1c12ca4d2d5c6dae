# full GPU suite + device-check run after k_rank_sel
O=gpurun_out/r02nn; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 900 python tools/sanitize.py > $O/sanitize.log 2>&1; echo "rc=$?" >> $O/sanitize.log
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "cluster_select" > $O/checks_paths.log 2>&1; echo "rc=$?" >> $O/checks_paths.log
