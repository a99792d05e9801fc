for n in base rg4 rg2 rg4p; do echo "== $n"; scripts/micro/sweep_trace_$n 1024 | head -4; scripts/micro/sweep_trace_$n 8192 | head -1; done
