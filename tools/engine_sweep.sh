BI_ENGINE_SKEW=3 timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_checkpoint.py -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do
for cfg in "0 4" "3 4" "3 2" "3 0"; do
set -- $cfg
BI_ENGINE_SKEW=$1 BI_PRIORITY_MODE=$2 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('skew $1 prio $2: ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2))"
done; done
BI_ENGINE_SKEW=3 BI_PRIORITY_MODE=4 python tools/engine_timeline.py 2>&1 | grep -E "run|^L" | cut -c1-250
