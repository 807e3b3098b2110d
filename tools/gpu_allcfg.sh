# bench lines for every BASELINE config (cfg 2 is the headline; the others are evidence)
mkdir -p gpurun_out
for c in 1 3 4 5; do
  st=5; [ $c = 5 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c rc=$?"; tail -c 600 gpurun_out/bench_cfg$c.err | tail -2
done
