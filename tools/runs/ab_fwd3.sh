for i in 1 2 3; do
  for L in paper_2211_03578_b200/libtlp.so "$@"; do
    echo -n "$(basename $L) "; TLP_LIB_PATH=$L timeout 120 python tools/time_fwd.py 10
  done
done
