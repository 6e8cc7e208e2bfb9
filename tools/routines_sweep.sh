for c in cfg3_syrk cfg3_syr2k cfg4_trmm cfg4_trsm; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('$c', 'e2e %.2f TF/s' % e['value'], '%.1f ms' % e['ms_per_step'], 'h2d %.2f GB' % (e['h2d_bytes_per_step']/1e9), 'launches', d['gpu_launches_e2e'])"
done
python tools/trace_e2e.py 16384 1024 16 2 4 2>&1 | head -2
