"""Timeline of a DAG schedule on the GPU (diagnostics): every launch stamped
when its dependencies are done and when its last kernel ended (HLU_STAMPS=1);
prints the measured critical path through the launch DAG, what it consists of,
graph scheduling gaps and the in-flight profile.
Usage: python tools/dag_timeline.py <case> [slot_us]"""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ["HLU_STAMPS"] = "1"
import numpy as np
import torch
import cases
from paper_1906_00874_b200 import ir, native_plan
from paper_1906_00874_b200.device import DeviceCall
from paper_1906_00874_b200.lowrank import TruncationControl
from paper_1906_00874_b200.planner import Layout


def main():
    name = sys.argv[1]
    slot = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
    build, ctl = cases.CASES[name]
    h, _ = build()
    L = Layout([h], cap=32, extra=[])
    nodes, index = native_plan.flatten_nodes(L)
    cmds = np.zeros(1, dtype=native_plan.CMD)
    cmds[0] = (native_plan.CMD_FACTOR, index[id(h)], 0, 0, 0, 0, 0, 0, 0, 0)
    p, _ = native_plan._build(L, nodes, cmds, native_plan.SPLIT_ROWS, dag_slot_ns=int(slot * 1000))
    call = DeviceCall(L, p, TruncationControl(*ctl), use_graph=True)
    call.snapshot()
    for r in range(2):
        call.restore()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(call.stream); call.launch(); e1.record(call.stream); call.sync()
        print(f"run {r}: {e0.elapsed_time(e1):.2f} ms (stamped graph)")
    call.check_errors()
    n = int(call.lib.hlu_schedule_stamps(call.handle, None))
    st = np.zeros(n, dtype=np.uint64)
    call.lib.hlu_schedule_stamps(call.handle, st.ctypes.data)
    st = st.astype(np.int64).reshape(-1, 2)
    nl = len(p.launches)
    ready, end = st[:nl, 0].astype(np.float64), st[:nl, 1].astype(np.float64)
    t0 = ready.min()
    ready = (ready - t0) / 1e3
    end = (end - t0) / 1e3  # us
    dur = end - ready
    Ls = p.launches
    kind = Ls["kind"].astype(np.int64)
    # truncation classes from the descriptors
    cls = kind.copy()
    names = {0: "getrf", 1: "trsm", 2: "gemm", 5: "gemmw", 3: "rkt-small", 6: "rkt-mid", 7: "rkt-merge"}
    for l in np.nonzero(kind == ir.K_RKT32)[0]:
        d = p.rkt[int(Ls[l]["first"])]
        cls[l] = 7 if int(d["part_count"]) > 2 else (3 if max(int(d["m"]), int(d["n"])) <= 64 else 6)
    ptr, idx = p.dag_ptr, p.dag_idx
    cp = np.zeros(nl)
    via = np.full(nl, -1, dtype=np.int64)
    gap = np.zeros(nl)
    for l in range(nl):
        d = idx[ptr[l]:ptr[l + 1]]
        if len(d):
            k = int(d[np.argmax(end[d])])
            gap[l] = ready[l] - end[k]
            j = int(d[np.argmax(cp[d])])
            cp[l] = cp[j]
            via[l] = k  # the predecessor that released it
        cp[l] += dur[l]
    wall = end.max()
    print(f"{name} slot {slot:g}us: launches {nl}, wall {wall / 1e3:.2f} ms, sum of launch durations {dur.sum() / 1e3:.1f} ms, "
          f"longest duration-weighted path {cp.max() / 1e3:.2f} ms")
    print(f"graph gaps (ready - last predecessor end): mean {gap.mean():.2f} us, p50 {np.percentile(gap, 50):.2f}, "
          f"p99 {np.percentile(gap, 99):.2f}, max {gap.max():.1f}")
    print("class        launches   ops    dur mean   p50    p90    max (us)   total ms")
    for c, nm in names.items():
        m = cls == c
        if m.any():
            print(f"{nm:11s} {m.sum():8d} {int(Ls['count'][m].sum()):8d} {dur[m].mean():8.1f} {np.percentile(dur[m], 50):7.1f} "
                  f"{np.percentile(dur[m], 90):7.1f} {dur[m].max():8.1f} {dur[m].sum() / 1e3:9.1f}")
    # the releasing chain that ends last: what actually bounded the run
    l = int(np.argmax(end))
    comp = {}
    gaps = 0.0
    hops = 0
    while l >= 0:
        c = names[int(cls[l])]
        a = comp.setdefault(c, [0, 0.0])
        a[0] += 1
        a[1] += dur[l]
        gaps += gap[l]
        hops += 1
        l = int(via[l])
    print(f"releasing chain of the last launch: {hops} launches, gaps {gaps / 1e3:.2f} ms; " +
          ", ".join(f"{k} {v[0]}/{v[1] / 1e3:.1f}ms" for k, v in comp.items()))
    # GEMM launches on that chain: serial tile steps of their longest CTA (static
    # dimension bounds: 64 x 64 output tiles, 32-deep k-steps, triple terms both products)
    g, t = p.gemm, p.terms

    def steps(rows, cols, inner):
        return -(-rows // 64) * -(-cols // 64) * -(-inner // 32)

    chain = []
    l = int(np.argmax(end))
    while l >= 0:
        chain.append(l)
        l = int(via[l])
    rows_out = []
    for l in chain:
        if int(kind[l]) not in (ir.K_GEMM, ir.K_GEMM_SMALL):
            continue
        f, c = int(Ls["first"][l]), int(Ls["count"][l])
        best, desc = 0, None
        for ch in range(f, f + c):
            tb, n = int(g["term_begin"][ch]), int(g["term_count"][ch])
            w = 0
            big = None
            for tm in t[tb:tb + n]:
                if tm["kind"] == ir.TERM_GEMM:
                    x = steps(int(tm["c"]["rows"]), int(tm["c"]["cols"]), int(tm["a"]["cols"]))
                elif tm["kind"] == ir.TERM_TRIPLE:
                    x = (steps(int(tm["m"]["rows"]), int(tm["c"]["cols"]), int(tm["m"]["cols"])) +
                         steps(int(tm["c"]["rows"]), int(tm["c"]["cols"]), int(tm["m"]["rows"])))
                else:
                    x = 0
                w += x
                if big is None or x > big[0]:
                    big = (x, int(tm["kind"]), int(tm["c"]["rows"]), int(tm["c"]["cols"]), int(tm["a"]["cols"]),
                           int(tm["m"]["rows"]), int(tm["m"]["cols"]))
            if w > best:
                best, desc = w, (n, big)
        rows_out.append((dur[l], best, c, desc))
    if rows_out:
        d = np.array([r[0] for r in rows_out])
        w = np.array([r[1] for r in rows_out], dtype=float)
        print(f"gemm launches on the chain: {len(d)}, duration mean {d.mean():.1f} us; serial tile steps of the longest "
              f"CTA: p50 {np.percentile(w, 50):.0f}, p90 {np.percentile(w, 90):.0f}, max {w.max():.0f}; "
              f"corr(duration, steps) {np.corrcoef(d, w)[0, 1]:.2f}; us per step (fit) {np.polyfit(w, d, 1)[0]:.2f}")
        for r in sorted(rows_out, key=lambda r: -r[0])[:12]:
            print(f"   dur {r[0]:8.1f} us, chains {r[2]:5d}, longest CTA {r[1]:5d} steps: terms {r[3][0]}, biggest term "
                  f"(steps, kind, Crows, Ccols, inner, Mrows, Mcols) {r[3][1]}")
    # in-flight profile
    ev = np.concatenate([np.stack([ready, np.ones(nl)], 1), np.stack([end, -np.ones(nl)], 1)])
    ev = ev[np.argsort(ev[:, 0], kind="stable")]
    infl = np.cumsum(ev[:, 1])
    dt = np.diff(ev[:, 0], append=ev[-1, 0])
    for lo, hi in ((0, 1), (1, 2), (2, 4), (4, 8), (8, 16), (16, 32), (32, 1 << 30)):
        m = (infl >= lo) & (infl < hi)
        print(f"  in flight [{lo},{hi}): {dt[m].sum() / 1e3:8.2f} ms")
    # ops per truncation launch
    m = kind == ir.K_RKT32
    c = Ls["count"][m]
    print("truncation launches by op count: " + ", ".join(
        f"<={b}: {int((c <= b).sum())}" for b in (1, 2, 4, 8, 16, 64, 256, 1 << 30)))
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"timeline_{name}_{slot:g}.npz"), ready=ready, end=end,
                        cls=cls, count=Ls["count"], ptr=ptr, idx=idx)


if __name__ == "__main__":
    main()
