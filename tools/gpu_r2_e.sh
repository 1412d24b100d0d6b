set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?"
for c in n3dv immersive stress; do timeout 300 python tools/ans_time.py $c 20 >> gpurun_out/r2e_ans.log 2>&1; done
timeout 900 bash tools/gpu_variants.sh n3dv bl_noskip bl_notsub bl_old > gpurun_out/r2e_var.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_decode_apply -c 1 -f -o gpurun_out/r2e_da_stress python tools/stage_times.py stress 1 > gpurun_out/r2e_da_ncu.log 2>&1; echo "ncu da rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_decode_apply -c 1 -f -o gpurun_out/r2e_da_n3dv python tools/stage_times.py n3dv 1 >> gpurun_out/r2e_da_ncu.log 2>&1; echo "ncu da rc=$?"
tail -n 3 gpurun_out/r2e_tests.log; cat gpurun_out/r2e_ans.log gpurun_out/r2e_var.log
