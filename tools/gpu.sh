#!/bin/bash
# Developer launcher for `gpurun -- bash tools/gpu.sh TASK [TASK ...]`; everything lands in gpurun_out/.
#   tests [PYTEST_ARGS]  GPU parity suite (pytest -m gpu), log in gpurun_out/pytest.log
#   smoke                __graft_entry__.smoke()
#   bench                default bench line + reference arm
#   launches             ncu launch list (gpu__time_duration, serialised) of a short bench run
#   ncu REGEX SKIP COUNT full ncu capture of codec_probe.py kernels matching REGEX (PINS env)
#   probe                codec_probe timings for every pin
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
while [ $# -gt 0 ]; do
  task=$1; shift
  case $task in
    tests)
      args=${PYTEST_ARGS:-"tests -m gpu -x -q"}
      timeout ${TEST_TIMEOUT:-1500} python -m pytest $args 2>&1 | tail -40 > gpurun_out/pytest.log
      tail -15 gpurun_out/pytest.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log ;;
    bench)
      timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
      timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
      cat gpurun_out/bench_ref.json ;;
    launches)
      timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
      python profiles/summarize_launches.py gpurun_out/launches.csv | head -20 ;;
    ncu)
      rx=$1; skip=$2; cnt=$3; shift 3
      PINS=${PINS:-auto} REPS=1 timeout 900 ncu --set full --import-source on --clock-control none \
        -k regex:"$rx" --launch-skip $skip --launch-count $cnt -o gpurun_out/prof_full -f \
        python tools/codec_probe.py > gpurun_out/ncu_prof.log 2>&1
      tail -3 gpurun_out/ncu_prof.log ;;
    probe)
      PINS=${PINS:-auto,fixedlen,raw,huffman} REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/probe.txt 2>&1
      cat gpurun_out/probe.txt ;;
    *) echo "unknown task $task" ;;
  esac
done
