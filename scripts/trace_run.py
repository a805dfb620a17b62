"""Per-warp timeline of one sampler launch (FM_LIB_VARIANT=trace build): when each warp found the
task queue exhausted and when it finished.  usage: FM_LIB_VARIANT=trace python scripts/trace_run.py cfg R"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_13230_b200 import fastmaxent as fm, workloads as WL
cfg = int(sys.argv[1]); R = int(sys.argv[2])
w = WL.workload(cfg)
x, y = WL.fitness(w)
plan = fm.sort_plan(torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda())
fn = fm.sample_ubcm if y is None else fm.sample_ecm
for _ in range(3):
    fn(plan, w.seed, n_samples=R).free()
fm.timing_enable(True); fm.timing_get(reset=True)
e = fn(plan, w.seed, n_samples=R); torch.cuda.synchronize()
t = fm.timing_get(reset=True)
tr = np.fromfile(os.environ.get("FM_TRACE_FILE", "/tmp/fm_trace.bin"), dtype=np.uint64).reshape(4096, 6)
tr = tr[tr[:, 0] > 0].astype(np.float64)
t0 = tr[:, 0].min()
start, done, end, it, itd, sm = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3, tr[:, 3], tr[:, 4], tr[:, 5]
print(f"cfg{cfg} R={R} kernel {t['sample_ms']:.3f} ms; warps {len(tr)}; span {end.max():.1f} us")
print("warp start us: max %.1f" % start.max())
print("queue exhausted (per warp) us: min %.1f p50 %.1f max %.1f" % (done.min(), np.median(done), done.max()))
print("warp end us: min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(end, [0, 10, 50, 90, 100])))
print("iterations per warp: p50 %d, after exhaustion p50 %d max %d" % (np.median(it), np.median(itd), itd.max()))
# active-warp profile over time
for q in np.linspace(0, end.max(), 21):
    print(f"  t={q:8.1f} us active warps {int(((start <= q) & (end > q)).sum()):5d}")
