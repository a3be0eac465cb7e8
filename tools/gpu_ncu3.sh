set -x
PINS=fixedlen REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^emit_kernel|fl_decode" -c 2 -o gpurun_out/fixed_full2 -f python tools/codec_probe.py > gpurun_out/ncu_full.log 2>&1
