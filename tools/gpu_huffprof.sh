# Huffman-pinned codec: timings, launch list and full ncu captures of the Huffman encode/decode kernels.
set -x
PINS=huffman REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/huff_probe.txt 2>&1
PINS=huffman REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/huff_launches.csv python tools/codec_probe.py > /dev/null 2>&1
PINS=huffman REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"emit_kernel|decode_kernel|scan_kernel" -s 3 -c 3 -o gpurun_out/huff_full -f python tools/codec_probe.py > gpurun_out/huff_ncu.log 2>&1
cat gpurun_out/huff_probe.txt; tail -3 gpurun_out/huff_ncu.log
