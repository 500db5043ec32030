python bench.py --no-e2e --no-cpu-baseline | python -c "
import json,sys
b=json.loads(sys.stdin.read())
print('headline', round(b['ms_per_step'],4), round(b['hbm_roofline_frac'],4))
for o in b['other_configs']: print(o['cfg'], round(o['ms_per_step'],4), round(o['hbm_roofline_frac'],4), o['l2'][:20])"
