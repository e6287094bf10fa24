timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_all_launches.csv python tools/time_train.py 1 > gpurun_out/train_all.stdout 2>&1
timeout 120 python tools/time_train.py 30
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "group_offsets or train_gemm" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_now.json 2> gpurun_out/bench_now.err; tail -c 600 gpurun_out/bench_now.json
