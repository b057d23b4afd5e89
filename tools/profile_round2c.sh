# Round-2 session-5 profiling pass (GPU box via gpurun): the launch list of the bench command itself
# (each ncu pass only after the same command exited 0 without ncu) and one ncu --set full capture of
# the leaf panel kernel at the cfg4 shape (64 blocks of 256) and at the cfg2 shape (8 blocks of 512).
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline"
$B > gpurun_out/s5_plain.json 2> gpurun_out/s5_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/s5_launches_bench.csv \
    $B > gpurun_out/s5_ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/s5_launches_bench.csv > gpurun_out/s5_launches_bench_summary.txt
python tools/profile_inv.py --n 256 --count 64 --reps 1 > gpurun_out/s5_inv64.txt 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:inv_panel -s 12 -c 1 -o gpurun_out/s5_k3_panel_64x256 \
    python tools/profile_inv.py --n 256 --count 64 --reps 1 > gpurun_out/s5_ncu_k3a.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:inv_panel -s 20 -c 1 -o gpurun_out/s5_k3_panel_8x512 \
    python tools/profile_inv.py --n 512 --count 8 --reps 1 > gpurun_out/s5_ncu_k3b.log 2>&1
for f in s5_k3_panel_64x256 s5_k3_panel_8x512; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null
done
tail -n 2 gpurun_out/s5_ncu_list.log gpurun_out/s5_ncu_k3a.log gpurun_out/s5_ncu_k3b.log
head -12 gpurun_out/s5_launches_bench_summary.txt
