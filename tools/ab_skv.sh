# Same-box A/B: config-4 local passes of one rank at P = 4 / 8 (cloud / P on one GPU), config 2.
for v in A B A B; do
  echo v=$v
  L=paper_2504_11729_b200/_lib/ab/lib$v.so
  for c in 32768 16384; do
    EP_LIB=$L python tools/splitkv_bench.py --batch 1 --cloud $c --steps 50 2>&1 | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    try: d=json.loads(l); print('skv', $c, round(d['local_attention_ms']*1000,2))
    except Exception: pass"
  done
  EP_LIB=$L python bench.py --no-extras --no-cpu-baseline --steps 3000 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', round(d['ms_per_step']*1000,2))"
done
