mkdir -p gpurun_out
PINS=huffman,auto REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/probe_new.txt 2>&1; cat gpurun_out/probe_new.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "huff or Huff or golden or codec" 2>&1 | tail -2
