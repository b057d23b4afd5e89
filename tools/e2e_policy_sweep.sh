# e2e (host-buffer) policy sweep: BI_PRIORITY_MODE / BI_RESERVE_SMS / BI_ENGINE_SKEW override both policies.
run() { env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"; }
run X=0
run BI_PRIORITY_MODE=1 BI_RESERVE_SMS=0
run BI_PRIORITY_MODE=4 BI_RESERVE_SMS=0
run BI_PRIORITY_MODE=4 BI_RESERVE_SMS=16
run BI_PRIORITY_MODE=1 BI_RESERVE_SMS=0 BI_ENGINE_SKEW=1
run BI_PRIORITY_MODE=1 BI_RESERVE_SMS=32
run BI_PRIORITY_MODE=3 BI_RESERVE_SMS=0
