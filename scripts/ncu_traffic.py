"""DRAM traffic per launch of one kernel family from an `ncu --set full` capture, next to the
algorithmic bytes of the same launches (profile records of the same run, launch order).

    python scripts/ncu_traffic.py --rep X.ncu-rep --records recs.json --kernel k_gemm [--M 3]
                                  [--update profiles/traffic.json]
"""
import argparse
import csv
import io
import json
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--records", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--M", type=int, default=0, help="only records summing M indices (0: any)")
    ap.add_argument("--update", default=None)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    launches = []
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
        launches.append({"name": d["Kernel Name"], "dram_read": rd, "dram_write": wr})
    recs = [r for r in json.load(open(args.records))
            if r["kernel"] == args.kernel and (args.M == 0 or r["step_end"] - r["step_begin"] == args.M)]
    n = min(len(launches), len(recs))
    pairs = []
    for L, R in zip(launches[:n], recs[:n]):
        pairs.append({"kernel": L["name"], "steps": [R["step_begin"], R["step_end"]],
                      "dram_bytes": L["dram_read"] + L["dram_write"], "algorithmic_bytes": R["bytes"]})
        print("%-60s steps %3d-%3d  DRAM %.3f GB  algorithmic %.3f GB  ratio %.3f" % (
            L["name"][:60], R["step_begin"], R["step_end"] - 1, (L["dram_read"] + L["dram_write"]) / 1e9,
            R["bytes"] / 1e9, (L["dram_read"] + L["dram_write"]) / R["bytes"]))
    dram = sum(p["dram_bytes"] for p in pairs) / n
    algo = sum(p["algorithmic_bytes"] for p in pairs) / n
    res = {"dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": algo,
           "dram_per_algorithmic_byte": dram / algo, "launches": pairs,
           "source": f"{args.rep}: dram__bytes_read.sum + dram__bytes_write.sum, mean over {n} captured launches"}
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}))
    if args.update:
        try:
            cur = json.load(open(args.update))
        except Exception:
            cur = {}
        if "bytes_per_algorithmic_byte" in cur:      # legacy single-kernel format
            cur = {}
        cur[args.kernel] = res
        json.dump(cur, open(args.update, "w"), indent=1)


if __name__ == "__main__":
    main()
