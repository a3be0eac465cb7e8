# Round-end evidence: GPU parity suite, smoke, default bench line, reference arm, bench launch list,
# full ncu of one Auto encode + decode call (2 warm-up calls x 6 kernels skipped).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
PINS=auto REPS=1 timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"range_kernel|emit_kernel|scan_kernel|profile_kernel|fl_decode|decode_kernel" \
  --launch-skip 12 --launch-count 6 -o gpurun_out/prof_full -f python tools/codec_probe.py > gpurun_out/ncu_prof.log 2>&1
tail -3 gpurun_out/pytest.log; cat gpurun_out/smoke.log gpurun_out/bench_final.json gpurun_out/bench_ref.json; tail -2 gpurun_out/ncu_prof.log
