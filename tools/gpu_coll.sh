set -x
timeout 900 python -m pytest tests/test_gpu_collectives_more.py tests/test_gpu_comm.py tests/test_gpu_multiproc.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_coll.log
cat gpurun_out/pytest_coll.log
