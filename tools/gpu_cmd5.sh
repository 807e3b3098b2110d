timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in 2 3 4; do
  timeout 120 python tools/run_cfg.py $c 2>&1 | tail -1
done
NYS_KM_NOBOUNDS=1 timeout 120 python tools/run_cfg.py 2 2>&1 | tail -1
