for c in cfg2 cfg3_syr2k cfg4_trmm; do for st in 4 8; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --streams $st 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('$c streams $st', 'e2e %.2f TF/s' % e['value'], '%.1f ms' % e['ms_per_step'])"
done; done
