"""Per-kernel warp-stall breakdown (pc sampling) and key throughput metrics from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines())); h = r[0]
cols = [i for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
extra = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
         "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]
for row in r[2:]:
    k = row[h.index("Kernel Name")][:30]
    tot = sum(float(row[i] or 0) for i in cols) or 1
    st = sorted(((h[i].split("stalled_")[1], 100 * float(row[i] or 0) / tot) for i in cols), key=lambda x: -x[1])
    print("==", k)
    print("   stalls:", ", ".join(f"{a} {b:.0f}%" for a, b in st if b >= 2))
    print("   ", {e.split("__")[1][:40]: row[h.index(e)] for e in extra if e in h})
