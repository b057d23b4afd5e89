timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x 2>&1 | tail -1
for c in 8 32; do python tools/profile_inv_graph.py --count $c; done; python tools/profile_inv_graph.py --count 64 --n 256
python tools/profile_inv.py --count 1 --n 5000 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b41.json 2> gpurun_out/b41.err; python -c "import json; d=json.load(open('gpurun_out/b41.json')); print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'e2e_ms', round(d['e2e']['ms_per_step'],2))"; done
