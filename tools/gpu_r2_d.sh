set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_entropy.py tests/test_gpu_parity.py tests/test_gpu_backward.py tests/test_gpu_mask.py -x -q -m gpu > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"
for c in n3dv immersive stress; do timeout 300 python tools/ans_time.py $c 20 >> gpurun_out/r2d_ans.log 2>&1; done
for c in n3dv meetroom immersive stress; do timeout 400 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2d_stages.log 2>&1; done
tail -n 3 gpurun_out/r2d_tests.log; cat gpurun_out/r2d_ans.log gpurun_out/r2d_stages.log
