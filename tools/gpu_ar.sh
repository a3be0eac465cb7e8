# Developer: the N=2 compressed AllReduce bench with both ranks on the one GPU (IPC loopback).
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_ar2.json 2> gpurun_out/bench_ar2.err
tail -3 gpurun_out/bench_ar2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_ar.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 1 --warmup 1 > /dev/null 2>&1
cat gpurun_out/bench_ar2.json
