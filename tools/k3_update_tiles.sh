# K3's K = 32 / 128 updates on other K1 tile paths: graph replay of the chain and engine device time.
for env in "BI_GEMM_TM=128" "BI_GEMM_TM=0 BI_GEMM_TM64_K=129 BI_GEMM_TM64_TILES=100000" "BI_GEMM_SMALL_TILES=200" "BI_GEMM_SMALL_TILES=300"; do
  echo "== $env"
  for spec in "64 256" "8 512" "32 512"; do set -- $spec; env $env python tools/profile_inv_graph.py --count $1 --n $2; done
  env $env python tools/engine_time.py | tr '\n' ' '; echo
done
