for d in 0 1 3 4; do
timeout 300 env TLP_TMA_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tma_gemm" -s 8 -c 8 --csv --log-file gpurun_out/tma_dbg$d.csv python tools/time_train.py 1 > /dev/null 2>&1
done
