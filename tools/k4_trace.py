"""Per-CTA timeline of the K4 score GEMM (EP_TRACE=1 path in kern_score.cu:
per CTA [start, first stage landed, last accumulator ready, scan done,
candidates done, end, first TMEM load, -] ns).

    EP_TRACE=1 EP_TRACE_SCORE_FILE=gpurun_out/k4.bin python tools/verify_bench.py --k 8 --steps 2 --warmup 1
    python tools/k4_trace.py gpurun_out/k4.bin
"""
import sys

import numpy as np


def main(path):
    t = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(-1, 8)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    s, f, a, sc, cd, e = [(t[:, i] - t0) / 1e3 for i in range(6)]
    p = lambda x: f"p50 {np.median(x):.1f} max {np.max(x):.1f}"
    print(f"CTAs {len(t)}: start spread {s.max():.1f} us; first stage landed {p(f - s)} us")
    print(f"  mainloop (first stage -> last accumulator ready) {p(a - f)} us")
    print(f"  scan {p(sc - a)} us; candidates {p(cd - sc)} us; end {p(e)} us")
    l0, wt = (t[:, 6] - t0) / 1e3, t[:, 7] / 1e3
    print(f"  acc ready -> first TMEM load {p(l0 - a)} us; waiting for staged partial chunks {p(wt)} us")
    order = np.argsort(e)[-5:]
    for i in order:
        print(f"  late CTA {i}: start {s[i]:.1f} first {f[i]:.1f} acc {a[i]:.1f} scan {sc[i]:.1f} end {e[i]:.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
