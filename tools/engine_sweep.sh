# Engine scheduling knobs on the bench workload (one line per setting).
for cfg in "148 16" "1000000 16" "1000000 0" "1000000 8" "148 16" "1000000 0"; do
set -- $cfg
BI_GEMM_SMALL_TILES=$1 BI_RESERVE_SMS=$2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('small-thr $1 reserve $2: ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'k1', round(d['roofline']['achieved'],2))"
done
