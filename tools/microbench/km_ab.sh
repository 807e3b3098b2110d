cat > /tmp/km_t.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_1901_06112_b200.landmarks import kmeans_device
from paper_1901_06112_b200.synthetic import CONFIGS
wl = CONFIGS[2]
f = torch.from_numpy(wl.image(seed=0)).cuda()
pts = f.reshape(3, -1)
for _ in range(3): r = kmeans_device(pts, 64, seed=0, max_iter=wl.max_iter)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); r = kmeans_device(pts, 64, seed=0, max_iter=wl.max_iter); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("iters", r.iterations, "ms", sorted(ts)[5], "errors", [round(e, 3) for e in r.errors[-4:]])
for it in (5, 8, 10, 12):
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); r2 = kmeans_device(pts, 64, seed=0, max_iter=it); b.record(); torch.cuda.synchronize()
    print("max_iter", it, "ms", round(a.elapsed_time(b), 3))
PY
python /tmp/km_t.py
NYS_KM_NOBOUNDS=1 python /tmp/km_t.py | head -1
