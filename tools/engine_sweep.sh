for cfg in 4 2 3 1 4; do
BI_ENGINE_LANES=$cfg python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('lanes $cfg: ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'k1', round(d['roofline']['achieved'],2))"
done
