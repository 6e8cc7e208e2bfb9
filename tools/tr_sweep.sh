for cfg in "8 1" "8 2" "16 2" "4 2" "16 3"; do set -- $cfg; echo "== chunk $1 tps $2"; python tools/trace_e2e.py 16384 1024 $1 $2 2>&1 | head -5; done
