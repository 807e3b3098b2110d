set -x
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench0.json 2> gpurun_out/s3/bench0.err; tail -c 600 gpurun_out/s3/bench0.json
bash tools/sanitize.sh s3/san
bash tools/prof_full.sh s3k2k3 "k_feat_hpass|k_vpass" 2
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
