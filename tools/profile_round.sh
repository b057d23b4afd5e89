# Round profiling pass (run on the GPU box from the repo root via gpurun).
mkdir -p gpurun_out
python tools/k1_traffic.py run > gpurun_out/t_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --nvtx --nvtx-include k1_phase/ --csv --log-file gpurun_out/k1_traffic.csv \
    python tools/k1_traffic.py run > gpurun_out/t_ncu.log 2>&1 && \
python tools/k1_traffic.py summarize gpurun_out/k1_traffic.csv gpurun_out/r01_ncu_gemm_summary.json > /dev/null
python tools/gemm_sweep.py --profile 2 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:gemm_tma -c 1 -o gpurun_out/r01_k1_tma_2048 \
    python tools/gemm_sweep.py --profile 2 > gpurun_out/p_ncu2.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r01_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
tail -2 gpurun_out/t_ncu.log gpurun_out/p_ncu*.log
