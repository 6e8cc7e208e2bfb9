# cfg4 TRSM e2e vs the leaf order (BX_TRSM_LEAF) and panel RHS width (BX_TRSM_RHS)
for cfg in "128 8" "128 16" "256 16" "256 32" "512 16" "512 32" "1024 16"; do set -- $cfg
  BX_TRSM_LEAF=$1 BX_TRSM_RHS=$2 BX_SWEEP="dict()" timeout 300 python tools/ramp_sweep.py trsm 16384 | sed "s/^/leaf $1 rhs $2: /"
done
