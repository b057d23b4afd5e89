# Does the 64x64 K1 tile help the small per-rank launches of the sharded engine?  (projection tool, P = 1, 4, 8)
run() { echo "== $*"; env "$@" python tools/shard_projection.py --ps 1,4,8 --reps 2 2>&1 | grep "^P="; }
run X=0
run BI_GEMM_TM=0
run BI_GEMM_TM=0 BI_GEMM_TM64_K=1000000 BI_GEMM_TM64_TILES=296
run BI_GEMM_TM=0 BI_GEMM_TM64_K=1000000 BI_GEMM_TM64_TILES=148
run BI_GEMM_TM=0 BI_GEMM_TM64_K=2048 BI_GEMM_TM64_TILES=600
run BI_GEMM_TM=0 BI_GEMM_TM64_K=1024 BI_GEMM_TM64_TILES=296
