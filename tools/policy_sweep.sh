run() { env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"; }
run X=1
run BI_PRIORITY_MODE=4
run BI_PRIORITY_MODE=4 BI_ENGINE_SKEW=1
run BI_ENGINE_SKEW=1
run BI_ENGINE_SKEW=2
run BI_ENGINE_LANES=2
run BI_PRIORITY_MODE=3
run BI_RESERVE_SMS=8
run BI_PRIORITY_MODE=0
run X=2
