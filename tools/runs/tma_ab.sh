# TMA GEMM A/B: building-block parity, train-step timing TLP_TMA_GEMM=1/0, launch list of one step
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "train_gemm_building_block" 2>&1 | tail -2
for v in 1 0 1 0; do TLP_TMA_GEMM=$v timeout 120 python tools/time_train.py 20; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tma_gemm|bimg" -s 16 -c 16 --csv --log-file gpurun_out/tma_launches.csv python tools/time_train.py 2 > /dev/null 2>&1
