set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mask.py tests/test_gpu_backward.py -x -q -m gpu --timeout 240 > gpurun_out/r2r_parity.log 2>&1; echo "parity rc=$?"
tail -n 3 gpurun_out/r2r_parity.log
for c in n3dv immersive meetroom stress; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2r_stages.log 2>&1; done
cat gpurun_out/r2r_stages.log
