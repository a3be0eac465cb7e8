# Round check: GPU parity suite, smoke, default bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err
tail -5 gpurun_out/pytest.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_default.json
