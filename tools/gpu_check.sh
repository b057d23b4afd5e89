timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do for c in 8 32; do python tools/profile_inv_graph.py --count $c; done; python tools/profile_inv_graph.py --count 64 --n 256; done
python tools/profile_inv.py --count 1 --n 5000 | tail -1
for i in 1 2; do python bench.py --steps 8 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('bench', round(d['value'],2), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"; done
