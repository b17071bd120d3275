# Same-box A/B of two library builds on the K3 128-row tile workloads.
for v in ${AB_VARIANTS:-A B A B}; do
  echo v=$v
  L=paper_2504_11729_b200/_lib/ab/lib$v.so
  EP_LIB=$L python tools/prefill_bench.py --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    try: d=json.loads(l); print('prefill', d['batch'], round(d['ms'],4), round(d['tflops']))
    except Exception: pass"
  EP_LIB=$L python tools/multitenant_bench.py 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mt', round(d['ms_per_step'],4))"
done
