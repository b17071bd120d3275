"""Debug: per-CTA timeline of the last K1 launch (EP_TRACE=1 build of the
trace buffer, see plan.cpp dump_trace): start / end, items, blocks, SM id and,
for the first 4 items of each CTA, the time its last block finished and the
time its item end (LSE combine, partial store, arrival, merge) finished.

    EP_TRACE=1 EP_TRACE_FILE=gpurun_out/k1.bin python tools/decode_only.py --steps 3
    python tools/k1_trace.py gpurun_out/k1.bin
"""
import sys

import numpy as np

NB = 1024


def main(path):
    raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
    se = raw[18 * NB:20 * NB].reshape(NB, 2)
    n = int((se[:, 0] > 0).sum())
    se = se[:n]
    wk = raw[20 * NB:22 * NB].reshape(NB, 2)[:n]
    ev = raw[22 * NB:30 * NB].reshape(NB, 4, 2)[:n]
    sm = raw[30 * NB:31 * NB][:n] if raw.size >= 31 * NB else np.zeros(n, np.int64)
    if raw.size >= 32 * NB:  # the epilogue warp may finish after the consumers
        ep_end = raw[31 * NB:32 * NB][:n]
        se = se.copy()
        se[:, 1] = np.maximum(se[:, 1], ep_end)
    t0 = se[:, 0].min()
    start = (se[:, 0] - t0) / 1e3
    end = (se[:, 1] - t0) / 1e3
    dur = end - start
    print(f"CTAs {n}: start spread {start.max():.2f} us; end min {end.min():.1f} p50 {np.median(end):.1f} "
          f"max {end.max():.1f} us")
    items = wk[:, 0]
    for k in sorted(set(items.tolist())):
        m = items == k
        print(f"  {k} items: {m.sum():3d} CTAs, end p50 {np.median(end[m]):.1f} max {end[m].max():.1f}, "
              f"blocks p50 {np.median(wk[m, 1]):.0f}, us/block p50 {np.median(dur[m] / wk[m, 1]):.3f}")
    # item ends
    costs = []
    for c in range(n):
        for i in range(min(4, items[c])):
            a, b = ev[c, i]
            if a > 0 and b > 0:
                costs.append((b - a) / 1e3)
    costs = np.array(costs)
    if costs.size:
        print(f"  item end (last block done -> item end done) us: p50 {np.median(costs):.2f} "
              f"p90 {np.percentile(costs, 90):.2f} max {costs.max():.2f}; total per CTA p50 "
              f"{np.median([sum((ev[c, i, 1] - ev[c, i, 0]) / 1e3 for i in range(min(4, items[c])) if ev[c, i, 0] > 0) for c in range(n)]):.2f}")
    # gap between item end and the next item's last-block time is the streaming
    order = np.argsort(end)
    print("  earliest:", [(int(c), round(float(end[c]), 1), int(items[c]), int(wk[c, 1]), int(sm[c])) for c in order[:6]])
    print("  latest:  ", [(int(c), round(float(end[c]), 1), int(items[c]), int(wk[c, 1]), int(sm[c])) for c in order[-6:]])
    # SM id correlation (GPC-ish: smid // 18)
    if sm.any():
        g = sm // 16
        for k in sorted(set(g.tolist())):
            m = g == k
            print(f"  smid {16 * k:3d}-{16 * k + 15:3d}: end mean {end[m].mean():.1f}, us/block {np.mean(dur[m] / wk[m, 1]):.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
