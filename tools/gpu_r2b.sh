set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cholesky" 2>&1 | tail -5
NYS_REFINE_TAU=0 NYS_REFINE_CERR=0 timeout 300 python tools/dump_out.py 3 norefine
