g++ -O3 -std=c++17 -ffp-contract=off -I include tools/microbench/host_plan.cpp -o /tmp/host_plan && python -c "
import numpy as np; np.load('gpurun_out/cfg2_centroids.npy').astype(np.float64).tofile('/tmp/cen.bin')" && /tmp/host_plan /tmp/cen.bin 64 3 0.1
lscpu | grep -E "Model name|^CPU\(s\)"
timeout 300 python tools/host_gap.py 2
