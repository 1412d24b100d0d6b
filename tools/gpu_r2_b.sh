# round 2 call b: changed-path tests, entropy decode timing, onesweep tile pass ncu (source level)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_entropy.py tests/test_gpu_densify.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?"
for c in n3dv immersive stress; do timeout 300 python tools/ans_time.py $c 20 >> gpurun_out/r2b_ans.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ans_decode -c 1 -f -o gpurun_out/r2b_ans python tools/ans_time.py n3dv 1 > gpurun_out/r2b_ans_ncu.log 2>&1; echo "ncu ans rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_onesweep32 -s 4 -c 2 -f -o gpurun_out/r2b_os python tools/stage_times.py n3dv 1 > gpurun_out/r2b_os_ncu.log 2>&1; echo "ncu os rc=$?"
tail -n 3 gpurun_out/r2b_tests.log; cat gpurun_out/r2b_ans.log
