"""Executed warp instructions and stall samples per source line of one kernel, from an ncu
`--page source --csv` export (SASS view) joined with `nvdisasm -g` line info of the same object.

    python scripts/ncu_source_lines.py <source.csv> <cubin> <mangled-kernel-prefix> [warp_tiles]
"""
import collections
import csv
import re
import subprocess
import sys


def main():
    src_csv, cubin, prefix = sys.argv[1:4]
    unit = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
    start = next(i for i, l in enumerate(dis) if l.startswith(".text." + prefix))
    end = next(i for i, l in enumerate(dis) if i > start and l.startswith("//--------------------- .text"))
    cur, amap = None, {}
    for l in dis[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+(.*?);", l)
        if m:
            amap[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(src_csv)))
    h = rows[1]
    ia, ie, iss = h.index("Address"), h.index("Instructions Executed"), h.index("# Samples")
    base = int(rows[2][ia], 16)
    per, samp = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        k = amap.get(int(r[ia], 16) - base)
        per[k] += int(r[ie])
        samp[k] += int(r[iss])
    tot, ts = sum(per.values()), sum(samp.values())
    print(f"kernel {rows[0][1]}\nexecuted warp instructions {tot} ({tot / unit:.1f} per unit of {unit:g}), stall samples {ts}")
    print("file:line | executed per unit | share | stall-sample share")
    for k, v in sorted(per.items(), key=lambda x: -x[1])[:40]:
        print(f"{k[0]}:{k[1]} | {v / unit:.1f} | {v / tot:.3f} | {samp[k] / ts:.3f}")


if __name__ == "__main__":
    main()
