# Engine scheduling knobs on the bench workload (one line per setting).
for cfg in 16 0 8 24 32 16 0; do
BI_RESERVE_SMS=$cfg python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('reserve $cfg: ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'k1', round(d['roofline']['achieved'],2))"
done
