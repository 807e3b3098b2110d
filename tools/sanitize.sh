# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_case.py;
# summaries -> gpurun_out/sanitize_*.txt (usage on the GPU box: bash tools/sanitize.sh)
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in blf nlm sync; do
    timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python tools/sanitize_case.py $case \
      > gpurun_out/sanitize_${tool}_${case}.txt 2>&1
    echo "$tool $case rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error|error' gpurun_out/sanitize_${tool}_${case}.txt | tail -2 | tr '\n' ' ')"
  done
done
