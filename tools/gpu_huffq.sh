# Huffman fast path: parity tests + timings + launch list.
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest.log
PINS=huffman,auto REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/huff_probe.txt 2>&1
PINS=huffman REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/huff_launches.csv python tools/codec_probe.py > /dev/null 2>&1
cat gpurun_out/pytest.log gpurun_out/huff_probe.txt
