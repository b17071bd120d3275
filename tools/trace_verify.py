"""Debug: EP_TRACE=1 EP_TRACE_FILE=gpurun_out/trace.bin python tools/trace_verify.py
then analyse the per-block clock64 events of CTA 0 of one verify launch."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import verify_bench
verify_bench.B = 64
print(verify_bench.run(4, 2, 1))
