mkdir -p gpurun_out
timeout 600 python tools/qsgd_probe.py > gpurun_out/qsgd_probe.txt 2>&1; tail -5 gpurun_out/qsgd_probe.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "qsgd or QSGD" 2>&1 | tail -2
