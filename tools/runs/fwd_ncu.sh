timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_forward -s 2 -c 1 -o gpurun_out/fwd_full python tools/time_fwd.py 1 > gpurun_out/fwd_ncu.log 2>&1
tail -3 gpurun_out/fwd_ncu.log
