"""Per-launch and per-family DRAM bytes and times from an `ncu --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X` list
(one C5a slice: scripts/c5a_one_pass.py).  Optionally records the k_gemm_hm family and its top launch
in profiles/traffic.json (bench.py's roofline.traffic).

    python scripts/ncu_family_dram.py gpurun_out/r4v/c5a_slice_dram.csv [--update profiles/traffic.json]
"""
import argparse
import collections
import csv
import json
import re

SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    iK, iM, iV, iU, iI = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        d = launches.setdefault(r[iI], {"kernel": r[iK]})
        d[r[iM]] = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1)
    return list(launches.values())


def family(name):
    m = re.search(r"tnb::(k_\w+)|(k_\w+)<", name)
    return (m.group(1) or m.group(2)) if m else name.split("(")[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--update", default=None)
    args = ap.parse_args()
    ls = load(args.csv)
    fam = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram": 0.0, "top": None})
    for d in ls:
        f = family(d["kernel"])
        if not f.startswith("k_"):
            continue
        dram = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        us = d.get("gpu__time_duration.sum", 0) * 1e6
        e = fam[f]
        e["launches"] += 1
        e["us"] += us
        e["dram"] += dram
        if e["top"] is None or us > e["top"]["us"]:
            e["top"] = {"kernel": d["kernel"][:80], "us": us, "dram_bytes": dram}
    for f, e in sorted(fam.items(), key=lambda kv: -kv[1]["us"]):
        print(f"{f:14s} launches {e['launches']:4d}  us {e['us']:9.1f}  DRAM {e['dram'] / 1e6:9.1f} MB  "
              f"top {e['top']['us']:.1f} us {e['top']['dram_bytes'] / 1e6:.1f} MB")
    if args.update:
        with open(args.update) as fh:
            tr = json.load(fh)
        e = fam.get("k_gemm_hm")
        if e:
            tr["k_gemm_hm"] = {"dram_bytes_per_launch": e["dram"] / e["launches"], "algorithmic_bytes_per_launch": None,
                               "top_launch": e["top"],
                               "source": f"{args.csv}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                                         "dram__bytes_write.sum over the prefix + one C5a slice (scripts/c5a_one_pass.py C5a 1)"}
        with open(args.update, "w") as fh:
            json.dump(tr, fh, indent=1)


if __name__ == "__main__":
    main()
