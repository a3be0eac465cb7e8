mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
PINS=huffman,auto REPS=10 timeout 300 python tools/codec_probe.py 2>&1 | tail -2
