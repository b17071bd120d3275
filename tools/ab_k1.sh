# Same-box A/B of two library builds (paper_2504_11729_b200/_lib/ab/lib{A,B}.so):
# config 2 decode, config 5 multi-tenant, config 3 verify, config 4 split-KV.
for v in A B A B; do
  echo v=$v
  L=paper_2504_11729_b200/_lib/ab/lib$v.so
  EP_LIB=$L python bench.py --no-extras --no-cpu-baseline --steps 3000 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  EP_LIB=$L python tools/multitenant_bench.py 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mt', round(d['ms_per_step'],4))"
  EP_LIB=$L python tools/verify_bench.py --steps 40 2>&1 | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    try: d=json.loads(l); print('verify', d['k'], round(d['step_p50_ms'],4), round(d['attention_p50_ms'],4))
    except Exception: pass"
done
