#!/bin/bash
# ncu evidence for one round (run under gpurun on ONE GPU; never multi-rank).
#   bash tools/profile_round.sh r01
# 1. launch list of one bench step (gpu__time_duration, --clock-control none)
# 2. --set full captures of the main kernels of the step
set -u
TAG=${1:-r01}
OUT=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $B > $OUT/${TAG}_launches.stdout 2>&1
for k in ${KERNELS:-tc_forward_kernel encode_warp_kernel topk_chunk_kernel rank_kernel tma_gemm_kernel tma_wgrad_kernel attn_bwd_tc_kernel attn_fwd_tc_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o $OUT/${TAG}_prof_$k $B > $OUT/${TAG}_prof_$k.log 2>&1
done
ls -la $OUT | grep $TAG
