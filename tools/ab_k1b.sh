# Same-box A/B: config 2 only (libA vs libB, extra env for B via ENVB)
for v in A B A B A B; do
  L=paper_2504_11729_b200/_lib/ab/lib$v.so
  if [ $v = B ]; then E="$ENVB"; else E="$ENVA"; fi
  r=$(env EP_LIB=$L $E python bench.py --no-extras --no-cpu-baseline --steps 3000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
  echo "$v $E cfg2 $r"
done
