# usage: bash tools/prof_full.sh tag 'kernel regex' count [bench args]
tag=$1; rx=$2; cnt=${3:-4}; shift 3
python bench.py --steps 1 --warmup 0 --no-cpu-baseline "$@" > gpurun_out/plainfull_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 0 --no-cpu-baseline "$@" > gpurun_out/ncufull_$tag.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncufull_$tag.log
