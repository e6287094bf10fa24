for i in 1 2; do timeout 120 python tools/time_train.py 30; TLP_PDL=0 timeout 120 python tools/time_train.py 30; done
timeout 300 python tools/gap_train.py 2>&1 | grep -v Warn | head -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
