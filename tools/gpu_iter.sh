mkdir -p gpurun_out
PINS=huffman REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k huff_emit_kernel --launch-skip 2 --launch-count 1 \
  -o /tmp/he -f python tools/codec_probe.py > gpurun_out/ncu_he.log 2>&1
ncu -i /tmp/he.ncu-rep --page source --csv --print-source=sass > gpurun_out/he_sass.csv 2>&1
ncu -i /tmp/he.ncu-rep --page raw --csv > gpurun_out/he_raw.csv 2>&1
tail -1 gpurun_out/ncu_he.log
