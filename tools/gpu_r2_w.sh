set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_entropy.py tests/test_gpu_first_frame.py -x -q -m gpu --timeout 240 > gpurun_out/r2w_t.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2w_t.log
for c in n3dv immersive meetroom stress; do timeout 300 python tools/ans_time.py $c 20 2>&1 | tail -1; done
