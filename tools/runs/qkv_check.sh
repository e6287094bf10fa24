timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "building_block" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train_large.py tests/test_gpu_nccl.py tests/test_gpu_lstm.py -q -x -k "grads or train or adam or nccl or finetune or mask or pos_enc or lstm" 2>&1 | tail -2
for i in 1 2; do timeout 120 python tools/time_train.py 20; done
TLP_TMA_GEMM=0 timeout 120 python tools/time_train.py 20
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 320 -c 80 --csv --log-file gpurun_out/step_launches.csv python tools/time_train.py 2 > /dev/null 2>&1
