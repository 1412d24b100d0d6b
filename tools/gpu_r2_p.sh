set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 240 > gpurun_out/r2p_parity.log 2>&1; echo "parity rc=$?"
tail -n 3 gpurun_out/r2p_parity.log
for c in n3dv stress; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2p_stages.log 2>&1; done
cat gpurun_out/r2p_stages.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_launches.csv python tools/stage_times.py n3dv 1 > gpurun_out/r2p_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/r2p_launches.csv 2>&1 | grep -i "piece\|emit\|total"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_emit$|k_piece_scatter" -c 2 -f -o gpurun_out/r2p_emit python tools/stage_times.py n3dv 1 > gpurun_out/r2p_ncu2.log 2>&1; echo "ncu2 rc=$?"
