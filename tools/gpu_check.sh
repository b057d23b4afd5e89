for cv in -1 100; do
echo "carveout $cv"
BI_CARVEOUT=$cv ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/k3_launches_$cv.csv python tools/profile_inv.py --count 8 --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/k3_launches_$cv.csv | head -5
for c in 8 32; do BI_CARVEOUT=$cv python tools/profile_inv.py --count $c; done 2>&1 | tail -2
BI_CARVEOUT=$cv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b26.json 2> gpurun_out/b26.err; python -c "import json; d=json.load(open('gpurun_out/b26.json')); print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'k1', round(d['roofline']['achieved'],2), 'gemm_ms', round(d['roofline']['kernel_ms_per_step'],2), 'leaf_ms', round(d['roofline']['leaf_inversion_ms_per_step'],2), 'e2e', round(d['e2e']['value'],2))"
done
