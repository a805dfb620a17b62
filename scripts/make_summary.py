"""Write profiles/<tag>_summary.md and profiles/traffic.json from a measurement run's artefacts
(profiles/<tag>_bench_*.json and the ncu raw exports).  usage: python scripts/make_summary.py r01_v10"""
import csv, json, os, sys

tag = sys.argv[1]
P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def raw(name):
    rows = list(csv.reader(open(os.path.join(P, f"{tag}_{name}_ncu_raw.csv"))))
    h, u, v = rows[0], rows[1], rows[-1]
    def get(k):
        x, unit = float(v[h.index(k)]), u[h.index(k)]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(unit, 1)
        return x * scale
    return get


b = {c: json.load(open(os.path.join(P, f"{tag}_bench_cfg{c}.json"))) for c in (2, 3, 4, 5)}
r = json.load(open(os.path.join(P, f"{tag}_bench_cfg3_refresh.json")))
ref = json.load(open(os.path.join(P, f"{tag}_bench_reference.json")))
d = json.load(open(os.path.join(P, f"{tag}_bench_default.json")))
U, E, K = raw("ksample"), raw("ksample_ecm"), raw("kcompact")
rd, wr = "dram__bytes_read.sum", "dram__bytes_write.sum"
json.dump({"k_sample": {
    "ubcm_cfg2": {"dram_read_bytes": int(U(rd)), "dram_write_bytes": int(U(wr)), "per": "launch (100 samples)",
                  "source": f"profiles/{tag}_ksample_ncu_raw.csv (ncu --set full, one launch)"},
    "ecm_cfg3": {"dram_read_bytes": int(E(rd)), "dram_write_bytes": int(E(wr)), "per": "launch (100 samples)",
                 "source": f"profiles/{tag}_ksample_ecm_ncu_raw.csv (ncu --set full, one launch)"}}},
          open(os.path.join(P, "traffic.json"), "w"), indent=1)


def row(c):
    x = b[c]; p = x["phase_ms_per_step"]; f = x["roofline"]
    return (f"| {c} | {x['config']['workload']} | **{x['value']:.3g}** | {x['proposals_per_s']:.3g} | {x['ms_per_step']:.3f} "
            f"({p['plan']:.3f} + {p['sample_kernel']:.3f} + {p['write']:.3f}) | **{f['frac']:.3f}** | "
            f"{x['cpu_baseline']['value']:.3g} ({x['cpu_baseline']['cores']} thr) | {x['e2e']['value']:.3g} |")


def m(get, k, scale=1.0, fmt="{:.0f}"):
    return fmt.format(get(k) * scale)


iss = "smsp__issue_active.avg.pct_of_peak_sustained_active"
l1, l2 = "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed"
L = [f"# Round 1 — final state ({tag}), all configs", "",
     f"Bench lines `{tag}_bench_cfg{{2,3,4,5}}.json` (config 2: 10 timed steps after 3 warm-up, configs 3–5: 5",
     f"steps; clocks in each line), `{tag}_bench_default.json` (the plain `python bench.py` line the driver runs:",
     f"{d['value']:.4g} edges/s, frac {d['roofline']['frac']:.3f}), `{tag}_bench_cfg3_refresh.json` (ECM with the",
     f"per-candidate β_min refresh) and `{tag}_bench_reference.json` (the reference arm = the CPU oracle).  GPU",
     f"tests: `{tag}_pytest.log`, `smoke()`: `{tag}_smoke.log`.", "",
     "| cfg | workload | accepted edges/s | proposals/s | ms per step (plan + sampler + write) | roofline.frac (k_sample) | CPU oracle edges/s | e2e edges/s (host buffers, PCIe) |",
     "|---|---|---|---|---|---|---|---|"] + [row(c) for c in (2, 3, 4, 5)] + [
     "", f"ECM with β_min refresh: {r['value']:.3g} edges/s, frac {r['roofline']['frac']:.3f}.  Reference arm (oracle, all host",
     f"cores, config 2): {ref['value']:.3g} edges/s.", "",
     f"ncu `--set full` of one launch (`{tag}_ksample_ncu_raw.csv` / `_details.csv` / SASS source page; ECM",
     f"`{tag}_ksample_ecm_ncu_*.csv`; compaction `{tag}_kcompact_ncu_raw.csv`):", "",
     "| | UBCM cfg 2 | ECM cfg 3 | k_compact cfg 2 |", "|---|---|---|---|",
     f"| duration (ncu, cold) | {U('gpu__time_duration.sum')*1e3:.3f} ms | {E('gpu__time_duration.sum')*1e3:.3f} ms | {K('gpu__time_duration.sum')*1e3:.3f} ms |",
     f"| DRAM read + write per launch | {U(rd)/1e6:.0f} MB + {U(wr)/1e6:.0f} MB (algorithmic output 800 MB) | {E(rd)/1e6:.0f} MB + {E(wr)/1e6:.0f} MB (algorithmic 900 MB) | {K(rd)/1e6:.0f} MB + {K(wr)/1e6:.0f} MB |",
     f"| issue active | {U(iss):.0f} % | {E(iss):.0f} % | — |",
     f"| L1 / L2 throughput | {U(l1):.0f} % / {U(l2):.0f} % | {E(l1):.0f} % / {E(l2):.0f} % | — |", "",
     f"Launch lists: `{tag}_launches.csv` (config 2) and `{tag}_launches_cfg4.csv` (config 4; cold and serialised:",
     f"compare shares).  Per-warp timeline: `{tag}_trace_cfg2.txt`.  The changes behind these numbers and the",
     "variants measured and rejected are in DESIGN.md §12."]
open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(L) + "\n")
print("\n".join(L[:16]))
