timeout 900 ncu --set full --clock-control none --import-source on -k regex:tma_gemm_kernel -s 40 -c 6 \
    -o gpurun_out/gemm_prof python tools/time_train.py 2 > gpurun_out/gemm_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 6 -c 2 \
    -o gpurun_out/attn_prof python tools/time_train.py 2 > gpurun_out/attn_prof.log 2>&1
ls -la gpurun_out
