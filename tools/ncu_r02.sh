# ncu --set full captures of the codec kernels (tools/codec_probe.py), summarised on the box:
# raw metrics CSV + per-instruction source page (SASS) per report; the .ncu-rep files are dropped
# (they exceed gpurun's copy-back limit).  Usage: bash tools/ncu_r02.sh TAG PINS REGEX COUNT
set -x
tag=$1; pins=$2; rx=$3; cnt=$4
mkdir -p gpurun_out
PINS=$pins REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$rx" \
  --launch-count $cnt -o /tmp/$tag -f python tools/codec_probe.py > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>&1
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>&1
gzip -f gpurun_out/${tag}_sass.csv
ls -la gpurun_out
tail -3 gpurun_out/ncu_$tag.log
