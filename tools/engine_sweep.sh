# Engine scheduling knobs on the bench workload (one line per setting).
for cfg in "1 2 16" "1 1 16" "2 1 16" "0 1 16" "1 1 0" "1 3 16"; do
set -- $cfg
BI_ENGINE_SKEW=$1 BI_PRIORITY_MODE=$2 BI_RESERVE_SMS=$3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('skew $1 prio $2 reserve $3: ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2))"
done
