mkdir -p gpurun_out/s3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench5.json 2> gpurun_out/s3/bench5.err; python -c "
import json;d=json.load(open('gpurun_out/s3/bench5.json'));print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['stage_ms'])"
for c in 1 3 4; do timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'],d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['stage_ms'])"; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
