# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_probe.py (a 3-rank loopback
# allreduce_eb, allgather, broadcast and one codec round trip); logs in gpurun_out/.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --target-processes all python tools/sanitize_probe.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
