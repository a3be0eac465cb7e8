# Loopback collective timings and an ncu launch list of one allreduce_eb (tools/group_probe.py).
set -x
mkdir -p gpurun_out
for p in auto fixedlen raw; do PIN=$p timeout 120 python tools/group_probe.py; done 2>&1 | tee gpurun_out/group.txt
ZC_RING_UNFUSED=1 timeout 120 python tools/group_probe.py 2>&1 | tee -a gpurun_out/group.txt
SHARED=1 timeout 120 python tools/group_probe.py 2>&1 | tee -a gpurun_out/group.txt
for nr in 4 8; do NR=$nr COUNT=$((32<<20)) timeout 120 python tools/group_probe.py; done 2>&1 | tee -a gpurun_out/group.txt
WARM=1 REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/coll_launches.csv python tools/group_probe.py > gpurun_out/ncu_coll.log 2>&1
tail -3 gpurun_out/ncu_coll.log
