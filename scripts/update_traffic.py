"""profiles/traffic.json from ncu raw-page exports: DRAM read / write bytes per launch of k_sample and of
the compaction kernel (bench.py's roofline.traffic / traffic_compact).

    python scripts/update_traffic.py TAG=CSV [TAG=CSV ...]     e.g. ubcm_cfg5=profiles/r02_v2_cfg5_..._raw.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "profiles", "traffic.json")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    tj = json.load(open(PATH)) if os.path.exists(PATH) else {}
    for arg in sys.argv[1:]:
        tag, path = arg.split("=", 1)
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        ir, iw, ik = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"), hdr.index("Kernel Name")
        for r in rows[2:]:
            kern = "k_sample" if "k_sample" in r[ik] else "k_compact" if "k_compact" in r[ik] else None
            if not kern:
                continue
            tj.setdefault(kern, {})[tag] = {
                "dram_read_bytes": int(float(r[ir]) * UNIT[units[ir]]),
                "dram_write_bytes": int(float(r[iw]) * UNIT[units[iw]]),
                "per": "launch",
                "source": f"{os.path.relpath(path, ROOT)} (ncu --set full, one launch; kernel {r[ik].split('(')[0][-24:]})",
            }
    json.dump(tj, open(PATH, "w"), indent=1)
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    main()
