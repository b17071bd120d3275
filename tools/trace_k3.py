"""Debug: clock64 trace of CTA 0 of the last K3 launch, for one of the K3
workloads, and a per-block breakdown of the steady state.

    EP_TRACE=1 EP_TRACE_FILE=gpurun_out/trace_k3.bin python tools/trace_k3.py {verify4|verify8|shared|prefill}
    python tools/trace_k3.py --analyse gpurun_out/trace_k3.bin
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

EV = ["KISSUE", "VISSUE", "QK", "PV", "S_SEEN", "P_DONE", "QK_START", "QK_FULLK", "QK_DONE",
      "PV_START", "PV_PFULL", "PV_DONE"]
NB = 1024


def analyse(path):
    raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
    t = raw[:18 * NB].reshape(18, NB)
    if raw.size >= 20 * NB:  # per-CTA globaltimer start / end (ns)
        se = raw[18 * NB:20 * NB].reshape(NB, 2)
        se = se[se[:, 0] > 0]
        t0 = se[:, 0].min()
        dur = (se[:, 1] - se[:, 0]) / 1e3
        end = (se[:, 1] - t0) / 1e3
        print(f"CTAs {len(se)}: start spread {(se[:, 0].max() - t0) / 1e3:.1f} us, "
              f"duration us min {dur.min():.1f} p50 {np.median(dur):.1f} max {dur.max():.1f}; "
              f"last end {end.max():.1f} us; slowest CTAs {np.argsort(-end)[:6].tolist()}")
        if raw.size >= 22 * NB:
            wk = raw[20 * NB:22 * NB].reshape(NB, 2)[:len(se)]
            order = np.argsort(-dur)
            print("  slowest (cta, us, items, blocks):",
                  [(int(c), round(float(dur[c]), 1), int(wk[c, 0]), int(wk[c, 1])) for c in order[:8]])
            print("  fastest (cta, us, items, blocks):",
                  [(int(c), round(float(dur[c]), 1), int(wk[c, 0]), int(wk[c, 1])) for c in order[-5:]])
            us_per_blk = dur / np.maximum(wk[:, 1], 1)
            print(f"  us per block p50 {np.median(us_per_blk):.3f}; items/CTA max {wk[:, 0].max()}")
    base = t[t > 0].min()
    n = int((t[4] > 0).sum())  # blocks with an S_SEEN event
    print(f"blocks traced: {n}")
    if n < 8:
        return
    lo, hi = n // 4, 3 * n // 4  # steady state
    s_seen, p_done = t[4, lo:hi], t[5, lo:hi]
    per = np.diff(s_seen)
    print(f"S_SEEN period p50 {np.median(per):.0f} cycles (mean {per.mean():.0f})")
    for name, a, b in (("softmax S_SEEN->P_DONE", 4, 5), ("QK issue->done", 6, 8), ("QK wait K", 6, 7),
                       ("PV start->done", 9, 11), ("PV wait P", 9, 10), ("P_DONE->PV_START", 5, 9),
                       ("QK_DONE->S_SEEN", 8, 4), ("KISSUE->QK_FULLK", 0, 7)):
        d = t[b, lo:hi] - t[a, lo:hi]
        d = d[(t[a, lo:hi] > 0) & (t[b, lo:hi] > 0)]
        if d.size:
            print(f"  {name:26s} p50 {np.median(d):7.0f}  mean {d.mean():7.0f}")
    print("total span", (t[t > 0].max() - base))


def items(path, n_show=24):
    """Per-item phases of CTA 0 (clock64): start -> Q in TMEM -> last PV
    done -> epilogue (O read) -> outputs stored -> end (merge)."""
    raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
    t = raw[:18 * NB].reshape(18, NB)
    st, qd, lp, ep, out, end = (t[12 + i] for i in range(6))
    n = int((st > 0).sum())
    print(f"items traced: {n}")
    print(" item  start->Q  Q->lastPV  lastPV->epi  epi->out  out->end  end->next start")
    for i in range(min(n, n_show)):
        nxt = st[i + 1] - end[i] if i + 1 < n else 0
        print(f"{i:5d} {qd[i]-st[i]:9d} {lp[i]-qd[i]:10d} {ep[i]-lp[i]:12d} {out[i]-ep[i]:9d} {end[i]-out[i]:9d} {nxt:9d}")
    tot = [np.median((b - a)[:n]) for a, b in ((st, qd), (qd, lp), (lp, ep), (ep, out), (out, end))]
    print("medians:", [int(x) for x in tot])


if __name__ == "__main__":
    if sys.argv[1] == "--analyse":
        analyse(sys.argv[2])
        sys.exit(0)
    if sys.argv[1] == "--items":
        items(sys.argv[2])
        sys.exit(0)
    kind = sys.argv[1]
    if kind.startswith("verify"):
        import verify_bench
        print(verify_bench.run(int(kind[6:]), 1, 1))
    elif kind == "decode":  # K1, config 2 (the trace of the last launch is kept)
        sys.argv = [sys.argv[0], "--steps", "3"]
        import decode_only
        decode_only.main()
    elif kind == "skv":  # K1, one rank's config-4 local pass (cloud tokens = argv[2])
        import splitkv_bench
        print(splitkv_bench.run(1, 3, 2, cloud=int(sys.argv[2])))
    elif kind == "shared":
        import multitenant_bench
        print(multitenant_bench.run(1, 1))
    else:
        import prefill_bench
        print(prefill_bench.run("cloud", 4, 1, 1))
