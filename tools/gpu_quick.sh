# Developer: fast-path parity tests + codec timings.
set -x
timeout 600 python -m pytest tests/test_gpu_codec.py -x -q -k "fixed_path or roundtrip_host or fused" 2>&1 | tail -25 > gpurun_out/pytest_quick.log
PINS=auto,fixedlen,raw,huffman REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/probe.txt 2>&1
ZC_NO_FIXED=1 PINS=auto REPS=10 timeout 300 python tools/codec_probe.py >> gpurun_out/probe.txt 2>&1
cat gpurun_out/pytest_quick.log gpurun_out/probe.txt
