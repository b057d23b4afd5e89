python tools/gemm_sweep.py --profile 2 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:gemm_tma -c 1 -o gpurun_out/r01_k1_tma_n64 python tools/gemm_sweep.py --profile 2 > gpurun_out/p_ncu2.log 2>&1
python tools/k1_traffic.py run > gpurun_out/t_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --nvtx --nvtx-include k1_phase/ --csv --log-file gpurun_out/k1_traffic.csv \
    python tools/k1_traffic.py run > gpurun_out/t_ncu.log 2>&1
tail -n 1 gpurun_out/p_ncu2.log gpurun_out/t_ncu.log
