#!/bin/bash
# A/B timing of the training step across libtlp builds: ROUNDS=3 tools/ab_train.sh a.so b.so ...
R=${ROUNDS:-3}
for i in $(seq $R); do
  for L in "$@"; do
    echo -n "$(basename $L): "; TLP_LIB_PATH=$L python tools/time_train.py 20
  done
done
