./tools/microbench/fir_tc 2>&1 | grep "N="
