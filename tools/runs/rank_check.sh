timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nccl.py -q -x -k "lambdarank or grads or adam or nccl" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_train_large.py -q -x 2>&1 | tail -2
for v in 1 0 1 0; do TLP_RANK_SPLIT=$v timeout 120 python tools/time_train.py 20; done
