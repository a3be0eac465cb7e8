set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest.log
PINS=huffman,auto REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/huff_probe.txt 2>&1
PINS=huffman REPS=1 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base function -k decode_kernel -c 1 -o gpurun_out/huff_dec -f python tools/codec_probe.py > gpurun_out/huff_ncu.log 2>&1
cat gpurun_out/pytest.log gpurun_out/huff_probe.txt; tail -3 gpurun_out/huff_ncu.log
