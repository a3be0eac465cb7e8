mkdir -p gpurun_out
PINS=huffman REPS=20 timeout 300 python tools/codec_probe.py > gpurun_out/probe_new.txt 2>&1; cat gpurun_out/probe_new.txt
