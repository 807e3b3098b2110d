"""Write a markdown summary of an ncu --set full report (per kernel: duration, DRAM traffic,
issue/FMA utilisation, top stall reasons) into profiles/."""
import csv, subprocess, sys

rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); h = r[0]; units = r[1]
def col(name):
    return h.index(name) if name in h else None
stall_cols = [i for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
keys = [("duration ms", "gpu__time_duration.sum"), ("DRAM read GB", "dram__bytes_read.sum"),
        ("DRAM write GB", "dram__bytes_write.sum"), ("DRAM BW % peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs/thread", "launch__registers_per_thread"), ("grid", "launch__grid_size"), ("block", "launch__block_size"),
        ("smem/block B", "launch__shared_mem_per_block_dynamic")]
lines = [f"# {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none). Durations are ncu-replayed "
         "(cold cache, serialised): compare shares, not absolutes.", "",
         "| kernel | " + " | ".join(k for k, _ in keys) + " | top stalls |", "|" + "---|" * (len(keys) + 2)]
for row in r[2:]:
    k = row[h.index("Kernel Name")].split("(")[0]
    vals = []
    for _, m in keys:
        i = col(m)
        v = row[i] if i is not None else ""
        if m.startswith("dram__bytes") and v:
            u = units[i]
            f = float(v.replace(",", ""))
            v = f"{f / (1e3 if u == 'Mbyte' else 1 if u == 'Gbyte' else 1e9 if u == 'byte' else 1e6 if u == 'Kbyte' else 1):.3f}"
        vals.append(v)
    tot = sum(float(row[i] or 0) for i in stall_cols) or 1
    st = sorted(((h[i].split("stalled_")[1], 100 * float(row[i] or 0) / tot) for i in stall_cols), key=lambda x: -x[1])[:4]
    lines.append(f"| {k} | " + " | ".join(vals) + " | " + ", ".join(f"{a} {b:.0f}%" for a, b in st) + " |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
