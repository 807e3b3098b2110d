"""Aggregate an ncu 'cuda,sass' source page to CUDA lines: stall samples (total or one reason) and instructions.
usage: ncu_src.py report.ncu-rep kernel_regex [top] [stall_column e.g. stall_long_sb]"""
import csv, subprocess, sys, collections

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
col = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.OrderedDict()
cur = None
h = None
for r in rows:
    if not r:
        continue
    if "Address" in r and "Warp Stall Sampling (All Samples)" in r:
        h = r
        continue
    if h is None:
        continue
    if len(r) >= 2 and r[0] and not r[0].startswith("0x"):
        cur = (r[0], r[1].strip()[:100])
        agg.setdefault(cur, [0, 0])
        continue
    if cur and len(r) == len(h):
        try:
            agg[cur][0] += int(float(r[h.index(col)] or 0))
            agg[cur][1] += int(r[h.index("Instructions Executed")] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"== {kern} [{col}]: samples {tot} instructions {toti}")
for (ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% {100*i/toti:5.1f}% instr  L{ln}: {src}")
