# usage: bash tools/gpu_check.sh  -- GPU tests, bench line, e2e paths
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d['e2e']['value'], d['e2e_reference_types']['value'])"
timeout 300 python bench.py --steps 5 --warmup 2 --sharded --no-cpu-baseline 2>/dev/null | grep metric | cut -c1-200
