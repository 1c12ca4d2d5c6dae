O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_stream.py tests/test_gpu_paths.py -q -x -k "batch or stream or cluster" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config F1 --steps 3 --warmup 5 --no-cpu > $O/f1.json 2>> $O/bench.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_batch -c 1 --csv --log-file $O/kbatch.csv python bench.py --config F1 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_il8.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --island-load 8 > $O/ncu2.log 2>&1
