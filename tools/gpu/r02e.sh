# gpurun script: GPU suite + C4 bench + island load 8 + ncu of the sparse pass
O=gpurun_out/r02e; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $O/bench.json 2>> $O/bench.err
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --island-load 8 > $O/il8.json 2>> $O/bench.err
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_fitness_sparse" --launch-skip 10 --launch-count 1 -o $O/sp python bench.py --steps 3 --warmup 12 --no-cpu --no-e2e > $O/ncu.log 2>&1
