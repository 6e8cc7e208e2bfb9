# e2e of every config under the default options vs the start-up ramp / deferred C off
export BX_SWEEP="dict();dict(ramp_tasks=0);dict(defer_c_move_in=False);dict(ramp_tasks=0,defer_c_move_in=False,first_chunk_steps=4);dict(ramp_chunk_steps=2);dict(ramp_tasks=16)"
timeout 300 python tools/ramp_sweep.py gemm 16384
timeout 300 python tools/ramp_sweep.py syrk 16384 8192
timeout 300 python tools/ramp_sweep.py syr2k 16384 8192
timeout 300 python tools/ramp_sweep.py trmm 16384
timeout 300 python tools/ramp_sweep.py trsm 16384
timeout 300 python tools/ramp_sweep.py symm 16384
