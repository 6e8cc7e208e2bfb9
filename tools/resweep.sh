# stream-count re-sweep per routine with the current kernels (auto = resolve_streams)
export BX_SWEEP="dict();dict(n_streams=8);dict(n_streams=12);dict(n_streams=16);dict()"
timeout 300 python tools/ramp_sweep.py syrk 16384 8192
timeout 300 python tools/ramp_sweep.py syr2k 16384 8192
timeout 300 python tools/ramp_sweep.py trmm 16384
timeout 300 python tools/ramp_sweep.py trsm 16384
