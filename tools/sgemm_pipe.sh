# tensor-pipe utilisation (clock-invariant) of the SGEMM kernels per variant and layout
BX_MNK=${BX_MNK:-16384,16384,16384} timeout 600 ncu --clock-control none -k regex:sgemm_tc \
  --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum \
  --csv python tools/sgemm_variants.py 16384 ${VARIANTS:-0 1} 2>/dev/null | python -c "
import csv, sys
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
iid = hdr.index('ID')
cur = {}
for r in rows[1:]:
    cur.setdefault(r[iid], {'k': r[ik]})[r[im]] = r[iv]
for i, d in cur.items():
    print(d['k'][:40], {k.split('.')[0].split('__')[1][:22]: v for k, v in d.items() if k != 'k'})
"
