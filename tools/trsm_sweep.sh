for leaf in 128; do
  BX_TRSM_LEAF=$leaf timeout 600 python bench.py --config cfg4_trsm --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('leaf $leaf', 'e2e %.2f TF/s' % e['value'], '%.1f ms' % e['ms_per_step'])"
done
