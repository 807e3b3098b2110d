timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lloyd or tensor_core" 2>&1 | tail -3
timeout 60 python tools/km_timing.py 4 | tail -1
NYS_KM_NOTC=1 timeout 60 python tools/km_timing.py 4 | tail -1
for c in 3; do timeout 100 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'],d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['stage_ms'])"; done
