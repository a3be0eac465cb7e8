set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest.log
PINS=auto,fixedlen REPS=10 timeout 300 python tools/codec_probe.py > gpurun_out/spec_probe.txt 2>&1
ZC_NO_SPEC=1 PINS=auto,fixedlen REPS=10 timeout 300 python tools/codec_probe.py >> gpurun_out/spec_probe.txt 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_spec.json 2> gpurun_out/bench_spec.err
tail -3 gpurun_out/pytest.log; cat gpurun_out/spec_probe.txt; python -c "import json; d=json.load(open('gpurun_out/bench_spec.json')); print(d['value'], d['ms_per_step'], d['eager_ms_per_step'], d['encode_ms'], d['decode_ms'], d['roofline'])"
