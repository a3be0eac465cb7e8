set -x
timeout 900 python -m pytest tests/test_gpu_collectives_more.py tests/test_gpu_comm.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_tl.log
timeout 300 python tools/timeline.py gpurun_out/timeline_r01.csv > gpurun_out/timeline_r01.json 2>&1
cat gpurun_out/pytest_tl.log gpurun_out/timeline_r01.json; head -5 gpurun_out/timeline_r01.csv
