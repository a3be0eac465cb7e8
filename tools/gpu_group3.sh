for ru in 4 8 16 32; do echo "region_units=$ru"; ZC_COMM_REGION_UNITS=$ru NR=2 python tools/group_probe.py; done
ZC_RING_KERNEL=1 NR=2 python tools/group_probe.py
