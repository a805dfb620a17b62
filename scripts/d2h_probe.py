"""Device->host bandwidth probe for the e2e leg: one cudaMemcpyAsync of B bytes into pinned
memory vs chunked copies over 1/2/4 streams (copy engines).  Prints one JSON line."""
import json
import sys

import torch

B = int(float(sys.argv[1])) if len(sys.argv) > 1 else 12_800_000_000
src = torch.empty(B, dtype=torch.uint8, device="cuda")
src.fill_(1)
dst = torch.empty(B, dtype=torch.uint8).pin_memory()
res = {"bytes": B}


def timeit(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


res["one_copy_gbs"] = B / timeit(lambda: dst.copy_(src, non_blocking=True)) / 1e6
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = 256 << 20

    def go():
        ev = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(ev)
        for i, o in enumerate(range(0, B, chunk)):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                dst[o:o + chunk].copy_(src[o:o + chunk], non_blocking=True)
        for s in streams:
            ev.wait_stream(s)
    res[f"chunked_{ns}streams_gbs"] = B / timeit(go) / 1e6
h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
res["h2d_1GiB_gbs"] = (1 << 30) / timeit(lambda: d.copy_(h, non_blocking=True)) / 1e6
print(json.dumps(res))
