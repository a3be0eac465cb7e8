# Round-2 (late) evidence on one B200 after the Huffman kernel changes; small outputs land in gpurun_out/
# (reports stay in /tmp on the box: gpurun copies back at most 64 MiB).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_final.log; cat gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; cat gpurun_out/bench_final.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
PINS=huffman REPS=1 timeout 900 ncu --set full --import-source on --clock-control none --launch-skip 12 --launch-count 6 \
  -o /tmp/r02_huffman -f python tools/codec_probe.py > gpurun_out/ncu_huff.log 2>&1
cp profiles/ncu_traffic.json /tmp/traffic_keep.json
python profiles/extract_ncu.py /tmp/r02_huffman.ncu-rep r02_huffman > /dev/null
ncu -i /tmp/r02_huffman.ncu-rep --page raw --csv > gpurun_out/r02_huffman_raw.csv 2>&1
cp /tmp/traffic_keep.json profiles/ncu_traffic.json   # the bench's traffic is the Auto call's
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
python profiles/summarize_launches.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches_summary.txt
cp profiles/r02_huffman_ncu_full_summary.txt gpurun_out/
du -sh gpurun_out
