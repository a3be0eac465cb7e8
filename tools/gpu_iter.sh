mkdir -p gpurun_out
PINS=huffman,auto REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/probe_new.txt 2>&1; cat gpurun_out/probe_new.txt
timeout 300 python -m pytest tests/test_gpu_codec.py -m gpu -x -q -k test_huffman_embedded_and_failures 2>&1 | grep -E "^E|assert|passed|failed" | head -20
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
