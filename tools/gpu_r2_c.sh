set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_entropy.py tests/test_gpu_densify.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
for c in n3dv immersive stress; do timeout 300 python tools/ans_time.py $c 20 >> gpurun_out/r2c_ans.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ans_decode -c 1 -f -o gpurun_out/r2c_ans python tools/ans_time.py n3dv 1 > gpurun_out/r2c_ans_ncu.log 2>&1; echo "ncu ans rc=$?"
tail -n 3 gpurun_out/r2c_tests.log; cat gpurun_out/r2c_ans.log
