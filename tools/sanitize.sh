# compute-sanitizer evidence for the hot-path kernels on small shapes.
# usage: bash tools/sanitize.sh [TAG]   (logs under gpurun_out/TAG/)
tag=${1:-san}; o=gpurun_out/$tag; mkdir -p $o
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/san_cases.py > $o/plain.log 2>&1 || { echo "plain run failed"; tail -5 $o/plain.log; }
for tool in memcheck racecheck synccheck initcheck; do
  for mode in 1 0; do   # in-stream plan (device gate on a host word) and the synchronous plan
    NYS_PIPELINED=$mode timeout 900 $CS --tool $tool --kernel-regex kns=nys --print-limit 40 \
      --log-file $o/${tool}_p$mode.log python tools/san_cases.py > $o/${tool}_p$mode.out 2>&1
    echo "$tool pipelined=$mode rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $o/${tool}_p$mode.log | tail -1)"
  done
done
# the SIMT K2 (ill-conditioned M fallback) under memcheck
NYS_K2_SIMT=1 NYS_PIPELINED=0 timeout 900 $CS --tool memcheck --kernel-regex kns=nys --print-limit 40 \
  --log-file $o/memcheck_simt.log python tools/san_cases.py blf > $o/memcheck_simt.out 2>&1
echo "memcheck simt rc=$? : $(grep 'ERROR SUMMARY' $o/memcheck_simt.log | tail -1)"
