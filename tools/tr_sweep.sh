for cfg in "16 2 0" "16 2 4" "16 2 2" "16 3 4"; do set -- $cfg; echo "== chunk $1 tps $2 first $3"; python tools/trace_e2e.py 16384 1024 $1 $2 $3 2>&1 | head -5; done
