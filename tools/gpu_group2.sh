for b in 2 4 8 16; do echo "banks=$b"; ZC_COMM_BANKS=$b NR=2 python tools/group_probe.py; done
