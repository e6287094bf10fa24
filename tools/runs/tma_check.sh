set -x

timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "train_gemm_building_block" 2>&1 | tail -5
for v in 1 0 1 0; do TLP_TMA_GEMM=$v timeout 120 python tools/time_train.py 20; done
timeout 600 python -m pytest tests/test_gpu_train_large.py tests/test_gpu_parity.py -q -x -k "grads or train" 2>&1 | tail -5
