#!/bin/bash
# A/B timing of libtlp builds on one box: ROUNDS=3 tools/ab_fwd.sh a.so b.so [c.so ...]
# (alternating processes so that clock / thermal drift hits every build equally)
R=${ROUNDS:-3}
for i in $(seq $R); do
  for L in "$@"; do
    echo -n "$(basename $L): "; TLP_LIB_PATH=$L python tools/time_fwd.py 10
  done
done
