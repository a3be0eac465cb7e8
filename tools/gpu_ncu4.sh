set -x
PINS=fixedlen REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"codec_kernel" -c 1 -o gpurun_out/codec_fl -f python tools/codec_probe.py > gpurun_out/ncu_full.log 2>&1
PINS=auto REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"codec_kernel" -c 1 -o gpurun_out/codec_auto -f python tools/codec_probe.py >> gpurun_out/ncu_full.log 2>&1
