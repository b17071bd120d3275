for v in A B A B; do echo v=$v; EP_LIB=paper_2504_11729_b200/_lib/ab/lib$v.so python bench.py --no-extras --no-cpu-baseline --steps 3000 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"ms_per_step\"]*1000,2), round(d[\"roofline\"][\"frac\"],4), d[\"clocks\"][\"sm_mhz\"])"; EP_LIB=paper_2504_11729_b200/_lib/ab/lib$v.so python tools/multitenant_bench.py 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"mt\", round(d[\"ms_per_step\"],4))"; EP_LIB=paper_2504_11729_b200/_lib/ab/lib$v.so python tools/splitkv_bench.py 2>&1 | python -c "
import json,sys
for l in sys.stdin.read().strip().splitlines():
    try: d=json.loads(l); print('skv', d['batch'], round(d['step_ms']*1000,1))
    except Exception: pass"; done
