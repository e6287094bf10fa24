#!/bin/bash
# ncu evidence for round 1 (run under gpurun; single GPU).
set -x
OUT=gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $OUT/launches_r01.csv $B > $OUT/launches_r01.stdout 2>&1
for k in tc_forward_kernel encode_kernel topk_chunk_kernel rank_kernel sgemm_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/prof_r01_$k $B > $OUT/prof_r01_$k.log 2>&1
done
ls -la $OUT
