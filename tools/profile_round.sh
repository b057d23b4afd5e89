mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
python tools/gemm_sweep.py --profile 2 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -c 1 -o gpurun_out/r01_k1_2048 python tools/gemm_sweep.py --profile 2 > gpurun_out/p_ncu2.log 2>&1
python tools/profile_inv.py --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:inv_panel -s 4 -c 1 -o gpurun_out/r01_k3_panel python tools/profile_inv.py --reps 1 > gpurun_out/p_ncu3.log 2>&1
for c in 8 32; do python tools/profile_inv.py --count $c; done > gpurun_out/p_inv.txt 2>&1
tail -3 gpurun_out/p_ncu*.log; cat gpurun_out/p_inv.txt
