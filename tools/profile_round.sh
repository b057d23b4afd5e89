# Round profiling pass (run on the GPU box from the repo root via gpurun).
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r01_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
python tools/profile_inv.py --count 8 --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:inv_panel -s 20 -c 1 -o gpurun_out/r01_k3_panel_final \
    python tools/profile_inv.py --count 8 --reps 1 > gpurun_out/p_ncu3.log 2>&1
./tools/microbench/panel_probe 512 8 > gpurun_out/panel_probe.txt 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -n 1 gpurun_out/p_ncu1.log gpurun_out/p_ncu3.log
