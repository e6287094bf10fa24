timeout 900 python -m pytest tests -q -x -m gpu -k "bf16 or forward or invariance or search or sharded or nccl or full_size or mask or pos_enc or dataset" 2>&1 | tail -2
bash tools/runs/ab_fwd3.sh tools/abl/nofold.so
