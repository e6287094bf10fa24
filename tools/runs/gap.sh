timeout 300 python tools/gap_train.py 2>&1 | tail -80
