set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_entropy.py -x -q -m gpu --timeout 240 > gpurun_out/r2g_parity.log 2>&1; echo "parity rc=$?"
tail -n 5 gpurun_out/r2g_parity.log
for c in n3dv stress; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2g_stages.log 2>&1; done
cat gpurun_out/r2g_stages.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches.csv python tools/stage_times.py n3dv 1 > gpurun_out/r2g_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/r2g_launches.csv 2>&1 | tail -40
