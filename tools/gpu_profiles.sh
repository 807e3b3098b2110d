# Round evidence on the GPU box: bench lines for every config, the reference arm, the cfg 2
# launch list and one ncu --set full capture of K2 / K3 / k_finish, full-size parity.
# usage: bash tools/gpu_profiles.sh TAG   (outputs under gpurun_out/TAG/)
tag=${1:-r2}; o=gpurun_out/$tag; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/reference_arm.json 2> $o/reference_arm.err
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $o/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/cfg2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $o/ncu_launch.log 2>&1
python tools/launches.py $o/cfg2_launches.csv > $o/cfg2_launches_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_seed_runs|k_lloyd_coop|k_feat_hpass|k_vpass|k_finish" -c 5 -o $o/cfg2_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $o/ncu_full.log 2>&1
for c in 1 2 3 4; do timeout 1200 python tools/fullsize_parity.py $c >> $o/fullsize_parity.jsonl 2>> $o/fullsize_parity.err; done
timeout 1200 python tools/fullsize_parity.py 5 1024 1024 >> $o/fullsize_parity.jsonl 2>> $o/fullsize_parity.err
ls -la $o
