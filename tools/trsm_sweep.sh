for cfg in "4 2" "8 2" "8 1" "6 2"; do set -- $cfg
  timeout 600 python bench.py --config cfg4_trsm --steps 2 --warmup 1 --no-cpu-baseline --streams $1 --tasks-per-stream $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('streams $1 tps $2', 'e2e %.2f TF/s' % e['value'], '%.1f ms' % e['ms_per_step'])"
done
