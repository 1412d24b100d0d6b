set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/r2bb_all.log 2>&1; echo "all rc=$?"; tail -n 3 gpurun_out/r2bb_all.log
for c in n3dv immersive meetroom stress; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2bb_stages.log 2>&1; done; cat gpurun_out/r2bb_stages.log
