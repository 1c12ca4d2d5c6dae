O=gpurun_out/r02ee; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config C3 --steps 500 --warmup 5 > $O/c3.json 2>> $O/bench.err
