# K3 outer-window width for the engine's leaf batches (graph-replayed latency) and its effect on the bench configs.
for rep in 1 2; do
for w in 128 256; do
  echo "== BI_GJ_WINDOW=$w (rep $rep)"
  for cfg in "256 64" "512 8" "512 32" "256 1" "128 64"; do
    read -r n cnt <<< "$cfg"
    BI_GJ_WINDOW=$w python tools/profile_inv_graph.py --n $n --count $cnt 2>&1 | tail -1
  done
done
done
for w in 128 256; do
  echo "== bench BI_GJ_WINDOW=$w"
  BI_GJ_WINDOW=$w python bench.py --steps 5 --warmup 3 --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('cfg4 ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'leaf', d['roofline']['leaf_inversion_ms_per_step'], 'pivotA', d['pivot_a_schedule']['ms_per_step'], 'cfg2', d['cfg2_batch']['eq7']['ms_per_batch'], d['cfg2_batch']['pivot_a']['ms_per_batch'], 'one', d['cfg2_batch']['one_matrix_e2e_ms'], 'res', d['residual_fro'])"
done
python tools/k3_fast_check.py 2>&1 | tail -3
BI_GJ_WINDOW=256 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -x -q 2>&1 | tail -2
