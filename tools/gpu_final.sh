# Round-end evidence: GPU parity suite, default bench line, bench launch list, Huffman-path ncu capture, QSGD probe.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest.log
timeout 400 python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
PINS=huffman REPS=1 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:"^(scan_kernel|huff_emit_kernel|decode_kernel)$" -c 3 -o gpurun_out/huff_final -f python tools/codec_probe.py > gpurun_out/huff_final.log 2>&1
timeout 600 python tools/qsgd_probe.py > gpurun_out/qsgd_probe.json 2>&1
tail -3 gpurun_out/pytest.log; cat gpurun_out/bench_final.json gpurun_out/bench_ref.json gpurun_out/qsgd_probe.json; tail -2 gpurun_out/huff_final.log
