# Developer: full ncu capture of the codec kernels (one launch each) + fp64 issue-rate probe.
set -x
./tools/fp64_rate > gpurun_out/fp64_rate.txt 2>&1
PINS=auto,huffman REPS=10 python tools/codec_probe.py > gpurun_out/probe.txt 2>&1
PINS=auto REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"emit_kernel|scan_kernel|decode_kernel|profile_kernel" -c 4 -o gpurun_out/codec_full -f python tools/codec_probe.py > gpurun_out/ncu_full.log 2>&1
PINS=huffman REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"emit_kernel|scan_kernel|decode_kernel" -c 3 -o gpurun_out/codec_huff_full -f python tools/codec_probe.py > gpurun_out/ncu_huff.log 2>&1
cat gpurun_out/probe.txt gpurun_out/fp64_rate.txt
