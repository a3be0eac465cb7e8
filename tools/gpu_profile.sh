# Round profile: full ncu of one Auto encode + decode call of the C1 workload (the 3rd call of
# tools/codec_probe.py: 2 warm-up calls x 9 kernels skipped), plus the bench launch list and line.
set -x
PINS=auto REPS=1 timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"range_kernel|emit_kernel|scan_kernel|profile_kernel|fl_decode|decode_kernel|fixup_kernel" \
  --launch-skip 18 --launch-count 9 -o gpurun_out/prof_full -f python tools/codec_probe.py > gpurun_out/ncu_prof.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err
tail -2 gpurun_out/ncu_prof.log; cat gpurun_out/bench_final.json
