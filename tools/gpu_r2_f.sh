set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 240 > gpurun_out/r2f_parity.log 2>&1; echo "parity rc=$?"
tail -n 30 gpurun_out/r2f_parity.log
for c in n3dv meetroom immersive stress; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2f_stages.log 2>&1; done
cat gpurun_out/r2f_stages.log
timeout 900 python -m pytest tests -q -m gpu --timeout 240 > gpurun_out/r2f_all.log 2>&1; echo "all rc=$?"; tail -n 8 gpurun_out/r2f_all.log
