for i in 1 2; do
python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('host mode 1 (default): e2e_ms', round(d['e2e']['ms_per_step'],2), 'ms', round(d['ms_per_step'],2))"
BI_PRIORITY_MODE=4 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('host mode 4: e2e_ms', round(d['e2e']['ms_per_step'],2), 'ms', round(d['ms_per_step'],2))"
done
