# Developer: encoder variants side by side.
for v in "ZC_TWO_PASS=1" "ZC_CODEC_LAG=2" "ZC_CODEC_LAG=6" "ZC_CODEC_LAG=12" "ZC_CODEC_LAG=24"; do
  echo "== $v"; env $v PINS=fixedlen,auto REPS=10 timeout 120 python tools/codec_probe.py 2>&1 | tail -2
done
