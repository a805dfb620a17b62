"""Sampler kernel time vs samples per call (tail overhead) and chunking knobs, config 2 or 3.
usage: python scripts/probe_tail.py [cfg]   (env FM_CHUNK_LANE_DRAWS / FM_CHUNK_FINE_DRAWS / FM_TAIL_FACTOR apply)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_13230_b200 import fastmaxent as fm, workloads as WL

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = WL.workload(cfg)
x, y = WL.fitness(w)
xd = torch.from_numpy(x).cuda()
yd = None if y is None else torch.from_numpy(y).cuda()
plan = fm.sort_plan(xd, yd)
fn = fm.sample_ubcm if y is None else fm.sample_ecm
fm.timing_enable(True)
tag = " ".join(f"{k}={os.environ[k]}" for k in ("FM_CHUNK_LANE_DRAWS", "FM_CHUNK_FINE_DRAWS", "FM_TAIL_FACTOR") if k in os.environ)
for R in (25, 50, 100, 200, 400):
    for _ in range(2):
        fn(plan, w.seed, n_samples=R).free()
    torch.cuda.synchronize()
    fm.timing_get(reset=True)
    n = 5
    edges = 0
    for _ in range(n):
        e = fn(plan, w.seed, n_samples=R)
        edges += e.n_edges
        e.free()
    torch.cuda.synchronize()
    t = fm.timing_get(reset=True)
    print(f"cfg{cfg} {tag} R={R:4d} kernel {t['sample_ms']/n:8.3f} ms  per-sample {t['sample_ms']/n/R*1000:7.2f} us  "
          f"write {t['write_ms']/n:7.3f} ms  edges/s(kernel) {edges/(t['sample_ms']/1000)/1e9:6.2f} G", flush=True)
