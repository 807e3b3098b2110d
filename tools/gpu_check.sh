# usage: bash tools/gpu_check.sh [tag]  -- gpu tests, short bench, launch list
tag=${1:-x}
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 300 python bench.py --steps 3 --warmup 2 --cpu-rows 16 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 1500 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
echo ncu rc=$?
