for g in 1 2 4 8 16; do
  dbg=$((g * 256))
  echo "group $g"
  BX_MNK=16384,16384,16384 BX_LAYOUTS=00 BX_SGEMM_DEBUG=$dbg timeout 300 ncu --clock-control none -k regex:sgemm_tc2p --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum -c 1 python tools/sgemm_variants.py 16384 2 2>/dev/null | grep -E "duration|per_second|pipe_tensor|dram"
done
for g in 2 4 8; do BX_MNK=32768,32768,32768 BX_LAYOUTS=00 BX_SGEMM_DEBUG=$((g*256)) timeout 300 python tools/sgemm_variants.py 32768 2 | sed "s/^/group $g: /"; done
