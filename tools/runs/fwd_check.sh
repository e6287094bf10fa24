timeout 900 python -m pytest tests -q -x -m gpu -k "bf16 or forward or invariance or search or sharded or nccl or full_size or mask or pos_enc or smoke or dataset" 2>&1 | tail -2
for i in 1 2; do timeout 120 python tools/time_fwd.py 10; done
