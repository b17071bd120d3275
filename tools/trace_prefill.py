"""Debug: EP_TRACE=1 EP_TRACE_FILE=gpurun_out/trace_pre.bin python tools/trace_prefill.py
then analyse CTA 0's per-item events (tools/trace_items.py)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import prefill_bench
kind = sys.argv[1] if len(sys.argv) > 1 else "cloud"
print(prefill_bench.run(kind, 4 if kind == "cloud" else 32, 1, 1))
