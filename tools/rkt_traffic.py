"""Summarise an ncu --csv launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per launch) of tools/ncu_case.py:
per-kernel launch counts, total and share of time, DRAM bytes; and the
truncation family's DRAM traffic per launch group against its algorithmic
bytes -> profiles/<round>/rkt_traffic.json (read by bench.py).
Usage: python tools/rkt_traffic.py launches.csv case.json out_summary.txt out_traffic.json"""
import csv
import json
import re
import sys
from collections import defaultdict


def main():
    path, case_json, out_txt, out_json = sys.argv[1:5]
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    rd = csv.reader(lines)
    hdr = next(rd)
    ix = {n: i for i, n in enumerate(hdr)}
    per = defaultdict(lambda: defaultdict(float))  # (id) -> metric -> value
    names = {}
    for r in rd:
        if len(r) < len(hdr):
            continue
        kid = int(r[ix["ID"]])
        names[kid] = r[ix["Kernel Name"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        m = r[ix["Metric Name"]]
        if m == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(unit, 1.0)  # -> us
        else:
            v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        per[kid][m] = v
    fam = defaultdict(lambda: [0, 0.0, 0.0])
    groups_seen = 0
    last_group_start = None
    for kid in sorted(per):
        ms = per[kid]
        nm = re.sub(r"\(.*", "", names[kid])
        nm = re.sub(r"^void ", "", nm)
        if "k_rkt_classify" in nm:
            groups_seen += 1
            last_group_start = kid
    partial = len(sys.argv) > 5 and sys.argv[5] == "--partial"
    if partial and last_group_start is not None:  # the capture stopped inside the last group: drop it
        per = {k: v for k, v in per.items() if k < last_group_start}
        groups_seen -= 1
    for kid, ms in per.items():
        nm = re.sub(r"\(.*", "", names[kid])
        nm = re.sub(r"^void ", "", nm)
        f_ = fam[nm]
        f_[0] += 1
        f_[1] += ms.get("gpu__time_duration.sum", 0.0)
        f_[2] += ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
    total = sum(v[1] for v in fam.values())
    case = json.loads(open(case_json).read().strip().splitlines()[-1])
    groups = groups_seen if groups_seen else case["rkt_launches"]
    per_launch = case.get("rkt_alg_bytes_per_launch")
    alg = float(sum(per_launch[:groups])) if per_launch and groups_seen else case["rkt_alg_bytes"]
    with open(out_txt, "w") as o:
        o.write(f"# ncu launch list of tools/ncu_case.py {case['case']} (non-graph, serialised, cold cache): "
                f"{sum(v[0] for v in fam.values())} launches, {total / 1e3:.1f} ms"
                f"{' (first ' + str(groups) + ' truncation launch groups of ' + str(case['rkt_launches']) + ')' if partial else ''}\n")
        o.write(f"{'kernel':60s} {'launches':>9s} {'total ms':>10s} {'share':>7s} {'mean us':>9s} {'dram MB':>10s}\n")
        for nm, v in sorted(fam.items(), key=lambda kv: -kv[1][1]):
            o.write(f"{nm[:60]:60s} {v[0]:9d} {v[1] / 1e3:10.2f} {v[1] / total:7.3f} {v[1] / v[0]:9.1f} {v[2] / 1e6:10.1f}\n")
        rkt = [v for nm, v in fam.items() if "k_rkt" in nm]
        t_rkt = sum(v[1] for v in rkt)
        d_rkt = sum(v[2] for v in rkt)
        if d_rkt > 0:
            o.write(f"\ntruncation family k_rkt_*: {t_rkt / 1e3:.1f} ms ({t_rkt / total:.3f} of the list), "
                    f"{groups} launch groups, dram {d_rkt / 1e6:.1f} MB = {d_rkt / groups / 1e3:.1f} kB per group; "
                    f"algorithmic {alg / 1e6:.1f} MB = {alg / groups / 1e3:.1f} kB per group; "
                    f"dram/algorithmic = {d_rkt / alg:.2f}\n")
    if d_rkt > 0 and out_json != "-":
        json.dump({"case": case["case"], "launch_groups": groups,
                   "dram_bytes_per_launch": d_rkt / groups, "alg_bytes_per_launch": alg / groups,
                   "dram_over_algorithmic": d_rkt / alg,
                   "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the k_rkt_* launches of a "
                             "non-graph factorization (tools/ncu_case.py), summed per truncation launch group"},
                  open(out_json, "w"))


if __name__ == "__main__":
    main()
