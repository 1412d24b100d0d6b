# Round-end evidence: bench lines for every config, the launch list of the bench command,
# and one ncu --set full capture of a frame's kernels (after the commands exit 0 without ncu).
set -u
R=${1:-r01}
mkdir -p gpurun_out
for c in n3dv tiny meetroom immersive stress; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_n3dv.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_" -s 67 -c 17 -f -o gpurun_out/${R}_full_n3dv \
  python tools/stage_times.py n3dv 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ans -c 2 -f -o gpurun_out/${R}_full_ans python tools/ans_time.py n3dv 1 > gpurun_out/ncu_ans.log 2>&1
echo "ans rc=$?"
