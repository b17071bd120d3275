# Same-box A/B of library builds on config 3 (verify step: K3 attention + K4 score / accept).
for v in ${AB_VARIANTS:-A B A B}; do
  L=paper_2504_11729_b200/_lib/ab/lib$v.so
  EP_LIB=$L python tools/verify_bench.py --steps 40 2>&1 | python -c "
import json,sys
out = []
for l in sys.stdin.read().strip().splitlines():
    try:
        d = json.loads(l)
    except Exception:
        continue
    out.append((d['k'], round(d['step_p50_ms'], 4), round(d['attention_p50_ms'], 4), round(d['score_accept_p50_ms'], 4)))
print('$v (k, step p50, attention, score+accept ms):', out)"
done
