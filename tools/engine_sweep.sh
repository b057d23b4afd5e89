for i in 1 2 3; do
python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('default(0,4): ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2))"
BI_ENGINE_SKEW=1 BI_PRIORITY_MODE=2 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('forced(1,2): ms', round(d['ms_per_step'],2))"
done
