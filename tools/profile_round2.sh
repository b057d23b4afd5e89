# Session-2 profiling pass (GPU box, repo root, via gpurun): bench line, bench launch list,
# ncu --set full of one engine K1 launch (bench phase) and of one K3 panel launch.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01s2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
python tools/k1_traffic.py run > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include k1_phase/ -k regex:gemm_tma_refill \
    -s 40 -c 1 -o gpurun_out/r01s2_k1_engine python tools/k1_traffic.py run > gpurun_out/p_ncu2.log 2>&1
python tools/profile_inv.py --count 8 --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:inv_panel -s 20 -c 1 -o gpurun_out/r01s2_k3_panel \
    python tools/profile_inv.py --count 8 --reps 1 > gpurun_out/p_ncu3.log 2>&1
tail -n 2 gpurun_out/p_ncu1.log gpurun_out/p_ncu2.log gpurun_out/p_ncu3.log
tail -n 1 gpurun_out/bench_final.json
