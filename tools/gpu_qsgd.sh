set -x
timeout 900 python -m pytest tests/test_gpu_qsgd.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_qsgd.log
timeout 600 python tools/qsgd_probe.py > gpurun_out/qsgd_probe.json 2>&1
cat gpurun_out/pytest_qsgd.log gpurun_out/qsgd_probe.json
