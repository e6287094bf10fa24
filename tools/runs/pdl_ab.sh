for i in 1 2 3 4; do timeout 120 python tools/time_train.py 100; TLP_PDL=0 timeout 120 python tools/time_train.py 100; done
