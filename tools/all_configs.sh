for c in cfg2 cfg3_syrk cfg3_syr2k cfg4_trmm cfg4_trsm; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('$c', 'value %.2f' % d['value'], 'e2e %.2f TF/s' % e['value'], '%.1f ms' % e['ms_per_step'], 'h2d %.2f GB' % (e['h2d_bytes_per_step']/1e9))"
done
