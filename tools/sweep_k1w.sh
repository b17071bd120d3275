# K1 item-weight sweep on config 2 / config 5 (same box): EP_K1_ITEM_WEIGHT = w blocks per item.
for w in ${WEIGHTS:-0 1 2 4 0 2}; do
  r=$(EP_K1_ITEM_WEIGHT=$w python bench.py --no-extras --no-cpu-baseline --steps 3000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
  m=$(EP_K1_ITEM_WEIGHT=$w python tools/multitenant_bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))")
  echo "w=$w cfg2 $r mt $m"
done
