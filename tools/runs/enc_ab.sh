timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -q -x -k "encode or crop or worked or fit or empty or search_round or full_size" 2>&1 | tail -2
for v in 0 1 0 1; do TLP_ENCODE_V1=$v timeout 120 python tools/time_encode.py; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:encode -s 3 -c 1 --csv --log-file gpurun_out/enc_launch.csv python tools/time_encode.py > /dev/null 2>&1
