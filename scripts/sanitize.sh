# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tests/sanitize_cases.py
# (every kernel family of the path on small inputs, results checked against the oracle).
# Logs: gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck racecheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "initcheck" ] && extra="--track-unused-memory no"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --target-processes all \
      python tests/sanitize_cases.py quick > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc $?"
  tail -3 gpurun_out/sanitize_$tool.log
done
