# cfg4 TRSM e2e vs the leaf order (BX_TRSM_LEAF) and panel RHS width (BX_TRSM_RHS)
for cfg in ${TRSM_CFGS:-128:8 128:16 256:16 256:32 512:16 512:32 1024:16}; do
  leaf=${cfg%:*}; rhs=${cfg#*:}
  BX_TRSM_LEAF=$leaf BX_TRSM_RHS=$rhs BX_SWEEP="dict()" timeout 300 python tools/ramp_sweep.py trsm 16384 | sed "s/^/leaf $leaf rhs $rhs: /"
done
