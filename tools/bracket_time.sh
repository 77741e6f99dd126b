# k_bracket_all duration (ncu, cold) for the current build at config 3
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bracket_all --csv $CMD 2>/dev/null | grep k_bracket | tail -2
