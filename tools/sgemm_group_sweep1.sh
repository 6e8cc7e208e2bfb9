# 2-SM SGEMM (variant 1): raster group vs DRAM traffic, clock and time (power-capped)
for g in 2 4 8 16 32; do
  echo "group $g"
  BX_MNK=16384,16384,16384 BX_LAYOUTS=00 BX_SGEMM_DEBUG=$((g * 256)) timeout 300 ncu --clock-control none -k regex:sgemm_tc2_ --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum -c 1 python tools/sgemm_variants.py 16384 1 2>/dev/null | grep -E "duration|per_second|dram"
done
for rep in 1 2; do for g in 4 8 16 32; do BX_MNK=32768,32768,32768 BX_LAYOUTS=00 BX_SGEMM_DEBUG=$((g*256)) timeout 300 python tools/sgemm_variants.py 32768 1 | sed "s/^/group $g: /"; done; done
