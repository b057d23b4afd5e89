for rep in 1 2; do
for w in 128 64 96 32; do
  echo "== BI_GJ_WINDOW=$w (rep $rep)"
  for cfg in "256 64" "512 8" "512 32" "256 1"; do
    read -r n cnt <<< "$cfg"
    BI_GJ_WINDOW=$w python tools/profile_inv_graph.py --n $n --count $cnt 2>&1 | tail -1
  done
done
done
for w in 64 96; do BI_GJ_WINDOW=$w python tools/k3_fast_check.py 2>&1 | tail -1; BI_GJ_WINDOW=$w python tools/k3_time.py 64x256 8x512 3x300; done
