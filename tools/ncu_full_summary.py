"""Per-kernel summary of an `ncu --set full` capture exported with
`ncu -i x.ncu-rep --page raw --csv`: duration, grid, registers, SM / fp64-pipe /
tensor-fp64 utilisation, DRAM bytes, active warps and the top sampled stall reasons.
Usage: python tools/ncu_full_summary.py raw.csv out.txt"""
import csv
import re
import sys
from collections import defaultdict


def f(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    groups = defaultdict(list)
    for r in data:
        nm = re.sub(r"\(.*", "", r[ix["Kernel Name"]])
        groups[nm].append(r)
    out = ["# ncu --set full --clock-control none, tools/ncu_case.py cfg3p_8192 (non-graph), launches 2000.. of the "
           "filtered kernels; means over the captured launches of each kernel\n"]
    cols = [("gpu__time_duration.sum", "dur"), ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
            ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%"),
            ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "dmma%"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
            ("dram__bytes_read.sum", "dramR"), ("dram__bytes_write.sum", "dramW")]
    for nm, rs in sorted(groups.items(), key=lambda kv: -sum(f(r[ix["gpu__time_duration.sum"]]) for r in kv[1])):
        line = f"{nm[:40]:40s} n={len(rs):2d}"
        for c, lab in cols:
            if c not in ix:
                continue
            v = sum(f(r[ix[c]]) for r in rs) / len(rs)
            u = units[ix[c]]
            line += f" {lab} {v:.4g}{u if lab in ('dur', 'dramR', 'dramW') else ''}"
        st = defaultdict(float)
        for r in rs:
            for s in stalls:
                st[s.replace("smsp__pcsamp_warps_issue_stalled_", "")] += f(r[ix[s]])
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
        line += " | stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top)
        out.append(line + "\n")
    open(sys.argv[2], "w").writelines(out)


if __name__ == "__main__":
    main()
