mkdir -p gpurun_out
PINS=huffman REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"::decode_kernel" --launch-skip 2 --launch-count 1 -o gpurun_out/huff_dec3 -f python tools/codec_probe.py > gpurun_out/ncu_dec3.log 2>&1; tail -2 gpurun_out/ncu_dec3.log
