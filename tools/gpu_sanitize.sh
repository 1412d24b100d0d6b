set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in tiny small; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $cfg > gpurun_out/san_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' gpurun_out/san_${tool}_${cfg}.log | tr '\n' ' ')"
  done
done
