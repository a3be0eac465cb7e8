NR=2 python tools/group_probe.py
NR=4 COUNT=$((32<<20)) python tools/group_probe.py
NR=2 REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_group.csv python tools/group_probe.py > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/launches_group.csv | head -20
