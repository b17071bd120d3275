"""Print the K9 rollout timings and per-stage barrier trace gathered by tools/run_k9.sh."""
import glob, json, sys
import numpy as np
for f in sorted(glob.glob("gpurun_out/mb_*.json")):
    try:
        d = json.load(open(f))
        print(f, {k: round(v["ms_per_step"] * 1e3, 1) for k, v in d["rollout_device"].items()}, "us/step")
    except Exception:
        print(f, open(f).read()[-400:])
for f in sorted(glob.glob("gpurun_out/trace_persist_*.bin")):
    t = np.fromfile(f, dtype=np.uint64).reshape(8, 32).astype(np.int64)
    for s in (1, 2):
        r = t[s]; st = r[31]
        n = [int(x - st) for x in r[:31] if x]
        print(f, s, "barriers (ns):", n, "gaps:", np.diff([0] + n).tolist())
