timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b30.json 2> gpurun_out/b30.err; tail -3 gpurun_out/b30.err; python -c "import json; d=json.load(open('gpurun_out/b30.json')); print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'k1', round(d['roofline']['achieved'],2)); print(d['pivot_a_schedule'])"
for c in 8 32; do python tools/profile_inv.py --count $c; done 2>&1 | tail -2
python tools/bench_configs.py --skip cfg1,cfg3 2>&1 | grep -E "^cfg"
