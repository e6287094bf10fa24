timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -q -x -k "encode or crop or worked or fit or empty or search_round or full_size" 2>&1 | tail -2
for i in 1 2 3; do for L in paper_2211_03578_b200/libtlp.so tools/abl/enc_old.so; do echo -n "$(basename $L) "; TLP_LIB_PATH=$L timeout 120 python tools/time_encode.py; done; done
