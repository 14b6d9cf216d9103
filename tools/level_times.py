"""Per-launch GPU time inside the CUDA graph (HLU_STAMPS=1 device timestamps
between launches) and what the slowest levels contain (diagnostics)."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import numpy as np
    import torch

    import cases
    from paper_1906_00874_b200 import _native, ir
    from paper_1906_00874_b200.device import DeviceCall
    from paper_1906_00874_b200.hlu import plan_call
    from paper_1906_00874_b200.lowrank import TruncationControl

    name = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    build, ctl = cases.CASES[name]
    h, _ = build()
    L, pl = plan_call([h], [("factor", h)], 32)
    call = DeviceCall(L, pl, TruncationControl(*ctl), use_graph=True)
    lib = _native.lib()
    for _ in range(2):
        call.upload()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(call.stream)
        call.launch()
        e1.record(call.stream)
        call.sync()
        print("graph run ms", e0.elapsed_time(e1))
    call.check_errors()
    p = call.packed
    call.upload()
    dt = call.launch_times() * 1e6  # us per launch entry (incl. its stamp node)
    call.check_errors()
    log = call.log.cpu().numpy()
    kinds = ["getrf", "trsm", "gemm", "rkt", "rkt64", "gemmw"]
    tot = collections.defaultdict(lambda: [0, 0.0])
    for i, L_ in enumerate(p.launches):
        k = kinds[int(L_["kind"])]
        tot[k][0] += 1
        tot[k][1] += dt[i]
    print("total us", dt.sum())
    # per level: dense launches vs truncation launches (overlap potential)
    lvl = p.launches["level"].astype(np.int64)
    isr = p.launches["kind"] == ir.K_RKT32
    D = np.bincount(lvl, weights=np.where(isr, 0.0, dt), minlength=p.nlevels)
    R = np.bincount(lvl, weights=np.where(isr, dt, 0.0), minlength=p.nlevels)
    print(f"levels {p.nlevels}: sum dense {D.sum() / 1e3:.1f} ms, sum trunc {R.sum() / 1e3:.1f} ms, "
          f"sum max(dense, trunc) per level {np.maximum(D, R).sum() / 1e3:.1f} ms")
    for k, (c, t) in tot.items():
        print(f"{k:6s} launches {c:6d} total {t / 1e3:9.1f} ms avg {t / c:8.1f} us")
    # truncation phases inside the graph: starts = previous launch's end stamp
    rk_idx = [i for i, L_ in enumerate(p.launches) if int(L_["kind"]) == ir.K_RKT32]
    ends = np.cumsum(np.concatenate([[0], dt]))  # us from the first stamp
    ps = call.last_phase_stamps.astype(np.float64)
    base = None
    # concurrent branches: r8 | r16 from classify; A | Abig; then Bw | B32 | B64; C | Cbig after all three
    names = ["classify", "r8", "r16", "-", "A", "Bw", "B32", "B64", "C", "Abig", "Cbig", "join"]
    NPH = len(names)
    ph = np.zeros((len(rk_idx), NPH))
    for r, i in enumerate(rk_idx):
        a_end = max(ps[r, 4], ps[r, 9])
        b_end = max(ps[r, 5], ps[r, 6], ps[r, 7])
        ph[r, 1] = (ps[r, 1] - ps[r, 0]) * 1e-3
        ph[r, 2] = (ps[r, 2] - ps[r, 0]) * 1e-3
        ph[r, 4] = (ps[r, 4] - ps[r, 0]) * 1e-3
        ph[r, 9] = (ps[r, 9] - ps[r, 0]) * 1e-3
        for k in (5, 6, 7):
            ph[r, k] = (ps[r, k] - a_end) * 1e-3
        ph[r, 8] = (ps[r, 8] - b_end) * 1e-3
        ph[r, 10] = (ps[r, 10] - b_end) * 1e-3
        ph[r, 11] = (ps[r, 11] - max(ps[r, 8], ps[r, 10])) * 1e-3
        ph[r, 0] = dt[i] - (ps[r, 11] - ps[r, 0]) * 1e-3
    print("truncation phases inside the graph (us): total / mean / max  [classify = level - rest]")
    for k in range(NPH):
        print(f"  {names[k]:8s} {ph[:, k].sum() / 1e3:9.1f} ms  mean {ph[:, k].mean():8.1f}  max {ph[:, k].max():9.1f}")
    # mean phase breakdown per level-duration bucket, with op-class counts
    import collections as _c
    acc = _c.defaultdict(lambda: [0, np.zeros(NPH), np.zeros(4)])
    for r, i in enumerate(rk_idx):
        b = 1 << max(0, int(dt[i]).bit_length())
        L_ = p.launches[i]
        d = p.rkt[int(L_["first"]): int(L_["first"]) + int(L_["count"])]
        lg = d["log"].astype(np.int64)
        K = np.where(d["mode"] == 0, log[lg] + log[lg + 1], log[lg])
        mm = np.maximum(d["m"], d["n"])
        cls = np.array([((mm <= 64) & (K <= 16)).sum(), ((mm > 64) & (mm <= 512)).sum(), (mm > 512).sum(), len(d)])
        a = acc[b]
        a[0] += 1
        a[1] += ph[r]
        a[2] += cls
    print("bucket(us) levels | mean phase us: " + " ".join(names) + " | mean ops: small, mid(<=512), big, all")
    for b in sorted(acc):
        n_, t_, c_ = acc[b]
        print(f"  <= {b:6d} {n_:5d} | " + " ".join(f"{x:6.0f}" for x in t_ / n_) + " | " + " ".join(f"{x:7.1f}" for x in c_ / n_))
    # rkt launches: time vs content
    rk = [i for i, L_ in enumerate(p.launches) if int(L_["kind"]) == ir.K_RKT32]
    hist = collections.defaultdict(lambda: [0, 0.0])
    for i in rk:
        b = 1 << max(0, int(dt[i]) .bit_length())
        hist[b][0] += 1
        hist[b][1] += dt[i]
    print("rkt launch time histogram (us bucket: count, total ms)")
    for b in sorted(hist):
        print(f"  <= {b:8d}: {hist[b][0]:6d} {hist[b][1] / 1e3:9.1f}")
    rpos = {i: r for r, i in enumerate(rk_idx)}
    order = sorted(range(len(dt)), key=lambda i: -dt[i])[:top]
    for i in order:
        L_ = p.launches[i]
        kind, count, first = int(L_["kind"]), int(L_["count"]), int(L_["first"])
        desc = ""
        if kind == ir.K_RKT32:
            d = p.rkt[first:first + count]
            _, start = ir.rkt_items(d["m"], d["n"])
            lg = d["log"].astype(np.int64)
            K = np.where(d["mode"] == 0, log[lg] + log[lg + 1], log[lg])
            kk = log[lg + 2]
            mm = np.maximum(d["m"], d["n"])
            desc = (f"ops {count} items {int(start[-1])} small {int(((np.maximum(d['m'], d['n']) <= 64) & (K <= 32)).sum())} "
                    f"max(m,n) {mm.max()} K max {K.max()} mean {K.mean():.1f} #K>32 {(K > 32).sum()} "
                    f"kk max {kk.max()} mode1 {(d['mode'] == 1).sum()} parts max {d['part_count'].max()}\n"
                    f"        phases " + " ".join(f"{names[k]}={ph[rpos[i], k]:.0f}" for k in range(NPH)))
        else:
            desc = f"count {count}"
        print(f"launch {i:6d} {kinds[kind]:6s} {dt[i]:10.1f} us  {desc}")


if __name__ == "__main__":
    main()
