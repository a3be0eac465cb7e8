set -x
PINS=auto REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launch_auto.csv python tools/codec_probe.py > /dev/null 2>&1
PINS=auto REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"emit_kernel|range_kernel|fl_decode" -c 3 -o gpurun_out/fixed_full -f python tools/codec_probe.py > gpurun_out/ncu_full.log 2>&1
