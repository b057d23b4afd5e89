# Round-2 session-4 profiling pass (GPU box via gpurun): cfg4 launch list + per-launch DRAM bytes of one run,
# and one ncu --set full capture of the level-6 arrows K1 launch (fat 4-warp kernel).
mkdir -p gpurun_out
python tools/ncu_engine_range.py --cfg 4 > /dev/null 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/s4_launches_cfg4.csv \
    python tools/ncu_engine_range.py --cfg 4 > gpurun_out/s4_ncu_list.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_tma_refill -c 1 \
    -o gpurun_out/s4_k1_fat_l6 python tools/ncu_engine_range.py --cfg 4 --steps 64 64 > gpurun_out/s4_ncu_full.log 2>&1
tail -n 2 gpurun_out/s4_ncu_list.log gpurun_out/s4_ncu_full.log
