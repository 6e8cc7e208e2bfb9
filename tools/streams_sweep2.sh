# compute streams per GPU vs e2e for every routine (tasks_per_stream 2)
export BX_SWEEP="dict(n_streams=4);dict(n_streams=8);dict(n_streams=12);dict(n_streams=16)"
timeout 300 python tools/ramp_sweep.py gemm 16384
timeout 300 python tools/ramp_sweep.py syrk 16384 8192
timeout 300 python tools/ramp_sweep.py syr2k 16384 8192
timeout 300 python tools/ramp_sweep.py trmm 16384
timeout 300 python tools/ramp_sweep.py symm 16384
