# final build: full GPU suite, device checks, smoke, C4 default-window line
O=gpurun_out/r04f; mkdir -p $O
timeout 1800 python -m pytest tests/ -q -x -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
PGA_LIB=paper_1403_4099_b200/libpga_check.so timeout 900 python tools/sanitize.py > $O/sanitize.log 2>&1; echo "rc=$?" >> $O/sanitize.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $O/c4.json 2>> $O/bench.err
