"""Per-step host/device timing of the config-5 step (plan, sample, free) to locate timing jitter."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2509_13230_b200 import fastmaxent as fm
from paper_2509_13230_b200 import workloads as WL

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w = WL.workload(cfg)
x, y = WL.fitness(w)
xd = torch.from_numpy(x).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fm.timing_enable(True)
for k in range(12):
    flush.fill_(k)
    torch.cuda.synchronize()
    fm.timing_get(reset=True)
    t0 = time.perf_counter()
    plan = fm.sort_plan(xd)
    t1 = time.perf_counter()
    e = fm.sample_ubcm(plan, w.seed, n_samples=w.n_samples)
    t2 = time.perf_counter()
    e.free()
    t3 = time.perf_counter()
    plan.free()
    t4 = time.perf_counter()
    tm = fm.timing_get(reset=True)
    print(f"step {k}: host plan {1e3*(t1-t0):7.2f} sample {1e3*(t2-t1):7.2f} efree {1e3*(t3-t2):6.2f} pfree {1e3*(t4-t3):6.2f} ms | dev plan {tm['plan_ms']:7.3f} sample {tm['sample_ms']:7.3f} write {tm['write_ms']:6.3f}", flush=True)
