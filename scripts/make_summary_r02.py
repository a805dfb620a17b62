"""profiles/<tag>_summary.md for a round-2 evidence run (scripts/gpu/r02_final.sh), from the files it left:

    python scripts/make_summary_r02.py r02_v13

reads profiles/<tag>_bench_{default,cfg2,cfg3,cfg4,reference}.json, <tag>_cfg{5,2,3,4}_ncu_raw.csv (raw-page
exports of the ncu --set full captures), <tag>_launches_cfg{5,4}.csv and <tag>_pytest.log.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def bench(name):
    path = os.path.join(P, f"{tag}_bench_{name}.json")
    if not os.path.exists(path):
        return None
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


def ncu_rows(cfg):
    path = os.path.join(P, f"{tag}_cfg{cfg}_ncu_raw.csv")
    if not os.path.exists(path):
        return []
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, v, u in zip(hdr, r, units)} for r in rows[2:]]


def launch_shares(cfg):
    path = os.path.join(P, f"{tag}_launches_cfg{cfg}.csv")
    if not os.path.exists(path):
        return None
    hdr, L = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                v = v / 1e3 if d["Metric Unit"] == "ns" else (v * 1e3 if d["Metric Unit"] == "ms" else v)
                name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("fm::", "").replace("<unnamed>::", "")
                L.append((name, v))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in L:
        agg[k][0] += 1
        agg[k][1] += t
    tot = sum(v[1] for v in agg.values())
    return [(k, n, t, 100 * t / tot) for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])], len(L), tot


out = []
lines = {"5 (default)": bench("default"), "2": bench("cfg2"), "3": bench("cfg3"), "4": bench("cfg4")}
d = lines["5 (default)"]
clk = d["clocks"] if d else {}
tests = ""
pl = os.path.join(P, f"{tag}_pytest.log")
if os.path.exists(pl):
    tests = open(pl).read().strip().splitlines()[-1]
out += [f"# Round 2 — final measurements ({tag}, one B200, {clk.get('sm_mhz')} MHz, throttle reasons {clk.get('reasons')})", "",
        "Command per line: `python bench.py [--config N] --steps 10 --warmup 3` (default line: no flags).  "
        f"GPU tests: `{tests}` (`{tag}_pytest.log`); smoke: `{tag}_smoke.log`.  e2e: `fm_sort_plan` (host x) + "
        "`fm_sample_to_host` with page-locked host buffers.", "",
        "| config | edges/s | step ms | plan | k_sample | write | k_sample frac | call frac | e2e edges/s | e2e ms | launches/step |",
        "|---|---|---|---|---|---|---|---|---|---|---|"]
for name, b in lines.items():
    if not b:
        continue
    ph, rf = b["phase_ms_per_step"], b["roofline"]
    out.append(f"| {name} {b['config']['workload']} | {b['value']:.3e} | {b['ms_per_step']:.3f} | {ph['plan']:.3f} | "
               f"{ph['sample_kernel']:.3f} | {ph['write']:.3f} | {rf['frac']:.3f} | {rf['call']['frac']:.3f} | "
               f"{b['e2e']['value']:.3e} | {b['e2e'].get('ms_per_step', float('nan')):.1f} | {b.get('gpu_launches')} |")
r = bench("reference")
if r:
    cb = r["cpu_baseline"]
    out += ["", f"Reference arm (`--impl reference`: the CPU oracle on {cb['cores']} host cores, {cb['sample']}): "
            f"{r['value']:.3e} {r['unit']}."]
b2 = bench("default_box2")
if b2:
    out += ["", f"The e2e leg is PCIe-bound and varies with the box: the default line re-run on a second box (`{tag}_bench_default_box2.json`): "
            f"{b2['value']:.3e} edges/s, e2e {b2['e2e']['value']:.3e} edges/s, {b2['e2e']['ms_per_step']:.1f} ms per step "
            f"({b2['e2e']['d2h_gbs']:.1f} GB/s; first box: {d['e2e']['d2h_gbs']:.1f} GB/s)."]
if d:
    rf = d["roofline"]
    out += ["", f"Default line's roofline object: bound `{rf['bound']}`, achieved {rf['achieved']:.4g} of peak {rf['peak']:.4g} {rf['unit']} "
            f"(frac {rf['frac']:.3f}); DRAM traffic per k_sample launch {rf.get('traffic')}, per compaction launch {rf.get('traffic_compact')} "
            "(bytes, `profiles/traffic.json`)."]

out += ["", f"## ncu (`--set full --clock-control none`, one launch each; `{tag}_cfg{{5,2,3,4}}_ncu_raw.csv`)", "",
        "| config | kernel | ms | DRAM read | DRAM write | issue active % | lanes per instruction | L2 hit % | registers | FP64 pipe % | warps/scheduler | eligible |",
        "|---|---|---|---|---|---|---|---|---|---|---|---|"]


def g(row, key):
    v, u = row.get(key, ("", ""))
    return v, u


for cfg in (5, 2, 3, 4):
    for row in ncu_rows(cfg):
        kn = row["Kernel Name"][0].split("(")[0]
        kn = kn[kn.find("k_"):] if "k_" in kn else kn
        t, tu = g(row, "gpu__time_duration.sum")
        t = float(t) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(tu, 1.0) if t else float("nan")
        rd, wr = g(row, "dram__bytes_read.sum"), g(row, "dram__bytes_write.sum")

        def f(key, fmt="{:.1f}"):
            v = g(row, key)[0]
            return fmt.format(float(v)) if v else "-"
        out.append(f"| {cfg} | `{kn[:40]}` | {t:.3f} | {float(rd[0]):.3f} {rd[1]} | {float(wr[0]):.3f} {wr[1]} | "
                   f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active')} | {f('smsp__thread_inst_executed_per_inst_executed.ratio', '{:.2f}')} | "
                   f"{f('lts__t_sector_hit_rate.pct')} | {f('launch__registers_per_thread', '{:.0f}')} | "
                   f"{f('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active')} | {f('smsp__warps_active.avg.per_cycle_active', '{:.2f}')} | "
                   f"{f('smsp__warps_eligible.avg.per_cycle_active', '{:.2f}')} |")

kp = os.path.join(P, f"{tag}_cfg4_kpass_ncu_raw.csv")
if os.path.exists(kp):
    rows = list(csv.reader(open(kp)))
    row = {h: (v, u) for h, v, u in zip(rows[0], rows[2], rows[1])}
    t, tu = row["gpu__time_duration.sum"]
    t_us = float(t) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(tu, 1.0)
    rd, wr = row["dram__bytes_read.sum"], row["dram__bytes_write.sum"]
    out += ["", f"Radix pass on config 4 (`{tag}_cfg4_kpass_ncu_raw.csv`, one of the 8 `k_pass<16>` launches, 1e7 keys): {t_us:.1f} us, "
            f"DRAM read {float(rd[0]):.1f} {rd[1]}, write {float(wr[0]):.1f} {wr[1]}, issue active "
            f"{float(row['smsp__issue_active.avg.pct_of_peak_sustained_active'][0]):.1f} %, "
            f"{float(row['launch__registers_per_thread'][0]):.0f} registers."]

out += ["", "## Launch lists (ncu `gpu__time_duration.sum`, `bench.py --steps 2 --warmup 1`, serialised, cold cache: compare shares)"]
for cfg in (5, 4):
    ls = launch_shares(cfg)
    if not ls:
        continue
    rows, n, tot = ls
    out += ["", f"`{tag}_launches_cfg{cfg}.csv`: {n} launches, {tot / 1e3:.2f} ms of GPU time.", "",
            "| kernel | launches | total us | share % | us per launch |", "|---|---|---|---|---|"]
    for k, c, t, sh in rows[:10]:
        out.append(f"| `{k[:48]}` | {c} | {t:.1f} | {sh:.1f} | {t / c:.1f} |")
    b = lines["5 (default)"] if cfg == 5 else lines["4"]
    if b:
        ph = b["phase_ms_per_step"]
        s = ph["plan"] + ph["sample_kernel"] + ph["write"]
        out += ["", f"CUDA-event phases of the config-{cfg} bench line for comparison: plan {100 * ph['plan'] / s:.1f} %, sampler "
                f"{100 * ph['sample_kernel'] / s:.1f} %, write (scan + offsets + compaction) {100 * ph['write'] / s:.1f} %."]

open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
