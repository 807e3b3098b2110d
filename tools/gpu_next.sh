# §8(f) rows: gpu tests, measurement lines, launch list
tag=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -q -x -k "pca or nlm or rec or brute or metrics" 2>&1 | tail -5
timeout 600 python tools/bench_next.py --steps 10 --warmup 3 > gpurun_out/next_$tag.jsonl 2> gpurun_out/next_$tag.err; echo "bench_next rc=$?"; cat gpurun_out/next_$tag.jsonl; tail -3 gpurun_out/next_$tag.err
timeout 300 python tools/bench_next.py --steps 1 --warmup 1 > gpurun_out/next_plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/next_launches_$tag.csv python tools/bench_next.py --steps 1 --warmup 1 > gpurun_out/next_ncu_$tag.log 2>&1
echo "ncu rc=$?"
