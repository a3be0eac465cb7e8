mkdir -p gpurun_out
timeout 900 python tools/sweep.py --ranks 2 --sizes-mb 1 4 16 64 256 1024 --out gpurun_out/r02_sweep_n2 > gpurun_out/sweep_n2.log 2>&1; tail -3 gpurun_out/sweep_n2.log
timeout 900 python tools/sweep.py --ranks 4 8 --sizes-mb 1 16 256 --out gpurun_out/r02_sweep_n48 > gpurun_out/sweep_n48.log 2>&1; tail -3 gpurun_out/sweep_n48.log
timeout 300 python tools/latency_probe.py > gpurun_out/latency.txt 2>&1; tail -20 gpurun_out/latency.txt
