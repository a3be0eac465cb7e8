mkdir -p gpurun_out
PINS=huffman REPS=20 timeout 300 python tools/codec_probe.py 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q -k "huff or Huff or golden or codec or ring" 2>&1 | tail -1
