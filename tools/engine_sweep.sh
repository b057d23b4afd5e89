# Engine scheduling knobs on the bench workload (one line per setting).
for cfg in "16 2" "0 2" "8 2" "24 2" "32 2" "16 0" "48 2"; do
set -- $cfg
BI_RESERVE_SMS=$1 BI_PRIORITY_MODE=$2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('reserve $1 prio $2: ms', round(d['ms_per_step'],2), 'value', round(d['value'],2))"
done
