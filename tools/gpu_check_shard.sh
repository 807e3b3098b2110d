timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 2 --sharded --no-cpu-baseline 2>/dev/null | grep metric | cut -c1-300
timeout 300 python tools/host_profile.py sharded 2>&1 | grep "ms per call"
