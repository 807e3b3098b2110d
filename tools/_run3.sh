timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lloyd or cell_pruned or kmeans or seeding" 2>&1 | tail -3
timeout 100 python tools/km_timing.py 2 | tail -1; timeout 100 python tools/km_timing.py 1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['stage_ms'])"
