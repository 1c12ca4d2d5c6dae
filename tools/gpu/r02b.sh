# gpurun script: new path tests, ncu source capture of the sparse pass and breed in the bench window
mkdir -p gpurun_out/r02b
timeout 1200 python -m pytest tests/test_gpu_paths.py -q --durations=10 > gpurun_out/r02b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02b/pytest.log
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_fitness_sparse|k_breed2" --launch-skip 20 --launch-count 2 -o gpurun_out/r02b/sp python bench.py --steps 3 --warmup 12 --no-cpu --no-e2e > gpurun_out/r02b/ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r02b/ncu.log
