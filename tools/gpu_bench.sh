# full default bench + reference arm + launch list + ncu full of the top kernel
tag=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/benchref_$tag.json 2> gpurun_out/benchref_$tag.err; echo "ref rc=$?"; tail -c 1500 gpurun_out/benchref_$tag.json
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_feat_hpass_tc|k_vpass|k_lloyd_coop|k_seed_coop" -c 4 -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncufull_$tag.log 2>&1
echo "ncu full rc=$?"
