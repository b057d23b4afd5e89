#!/bin/bash
# A/B of K3 builds: each argument is an alternative .so (loaded via BI_LIB),
# compared with the in-tree library on graph-replayed K3 latency at the leaf shapes.
set -u
libs=("$@" "")
for rep in 1 2; do
  for lib in "${libs[@]}"; do
    echo "== lib ${lib:-in-tree} (rep $rep)"
    for cfg in "512 8" "512 32" "256 64"; do
      read -r n cnt <<< "$cfg"
      BI_LIB=$lib python tools/profile_inv_graph.py --n $n --count $cnt 2>&1 | tail -1
    done
  done
done
