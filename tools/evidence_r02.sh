# Round-2 evidence on one B200, everything copied into gpurun_out/ (then into profiles/ by hand):
#  1. ncu --set full of one Auto encode + decode call of the codec bench workload (6 launches) ->
#     r02_final_ncu_full_summary.txt + ncu_traffic.json (bench.py's roofline.traffic);
#  2. the same for the Huffman-pinned call -> r02_huffman_ncu_full_summary.txt;
#  3. the fused ring kernel and the staged kernels of a loopback allreduce_eb -> r02_ring_*;
#  4. the bench's launch list (gpu__time_duration, serialised).
set -x
mkdir -p gpurun_out
PINS=auto REPS=1 timeout 600 ncu --set full --clock-control none --launch-skip 12 --launch-count 6 \
  -o /tmp/r02_final -f python tools/codec_probe.py > gpurun_out/ncu_final.log 2>&1
python profiles/extract_ncu.py /tmp/r02_final.ncu-rep r02_final > /dev/null
PINS=huffman REPS=1 timeout 900 ncu --set full --clock-control none --launch-skip 12 --launch-count 6 \
  -o /tmp/r02_huffman -f python tools/codec_probe.py > gpurun_out/ncu_huff.log 2>&1
cp profiles/ncu_traffic.json /tmp/traffic_keep.json
python profiles/extract_ncu.py /tmp/r02_huffman.ncu-rep r02_huffman > /dev/null
cp /tmp/traffic_keep.json profiles/ncu_traffic.json   # the bench's traffic is the Auto call's
WARM=1 REPS=1 timeout 600 ncu --set full --clock-control none -k regex:"ring_fused|emit_kernel|fl_decode|profile_kernel" \
  --launch-skip 10 --launch-count 10 -o /tmp/r02_ring -f python tools/group_probe.py > gpurun_out/ncu_ring.log 2>&1
ZC_RING_NOFUSEDK=1 WARM=1 REPS=1 timeout 600 ncu --set full --clock-control none \
  -k regex:"emit_kernel|fl_decode|profile_kernel|range_kernel" --launch-skip 10 --launch-count 10 \
  -o /tmp/r02_staged -f python tools/group_probe.py > gpurun_out/ncu_staged.log 2>&1
for t in r02_ring r02_staged; do
  ncu -i /tmp/$t.ncu-rep --page raw --csv > gpurun_out/${t}_raw.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
python profiles/summarize_launches.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches_summary.txt
cp profiles/r02_final_ncu_full_summary.txt profiles/r02_huffman_ncu_full_summary.txt profiles/ncu_traffic.json gpurun_out/
tail -2 gpurun_out/ncu_final.log gpurun_out/ncu_huff.log gpurun_out/ncu_ring.log gpurun_out/ncu_staged.log
