# per-launch device times of one train step (TMA GEMM on), then ncu --set full of 4 TMA GEMM launches
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 120 --csv --log-file gpurun_out/tma_launches.csv python tools/time_train.py 2 > /dev/null 2>&1
timeout 300 env TLP_TMA_GEMM=0 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 120 --csv --log-file gpurun_out/bimg_launches.csv python tools/time_train.py 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_gemm -s 8 -c 4 -o gpurun_out/tma_full python tools/time_train.py 1 > /dev/null 2>&1
ls -la gpurun_out
