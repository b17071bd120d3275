"""Per-CTA timeline of the K4 score GEMM (EP_TRACE=1 build path in
kern_score.cu: [start, first stage landed, last MMA done, end] ns per CTA).

    EP_TRACE=1 EP_TRACE_SCORE_FILE=gpurun_out/k4.bin python tools/verify_bench.py --k 8 --steps 2 --warmup 1
    python tools/k4_trace.py gpurun_out/k4.bin
"""
import sys

import numpy as np


def main(path):
    t = np.fromfile(path, dtype=np.uint64).astype(np.int64).reshape(-1, 4)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    s, f, m, e = [(t[:, i] - t0) / 1e3 for i in range(4)]
    print(f"CTAs {len(t)}: start spread {s.max():.1f} us; first stage landed after p50 {np.median(f - s):.1f} us; "
          f"mainloop (first stage -> MMAs done) p50 {np.median(m - f):.1f} max {np.max(m - f):.1f} us; "
          f"epilogue p50 {np.median(e - m):.1f} max {np.max(e - m):.1f} us; end max {e.max():.1f} us")
    late = s > 1.0
    print(f"CTAs starting after 1 us (second wave / co-resident): {int(late.sum())}, their start p50 {np.median(s[late]) if late.any() else 0:.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
