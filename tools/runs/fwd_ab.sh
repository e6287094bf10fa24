# forward A/B: parity subset + score timing with env toggles ($1 = env var name)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py tests/test_gpu_nccl.py -q -x -k "bf16 or forward or invariance or search or sharded or nccl or full_size or mask or pos_enc" 2>&1 | tail -2
for v in 1 0 1 0 1 0; do env $1=$v timeout 120 python tools/time_fwd.py; done
