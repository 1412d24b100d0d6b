# Round-2 evidence: GPU suite, bench lines + launch list + ncu captures (gpu_profile_round.sh),
# and the --as-rank predictions of the multi-GPU table
set -u
mkdir -p gpurun_out
R=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${R}_tests.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/${R}_tests.log
bash tools/gpu_profile_round.sh $R
for c in n3dv immersive meetroom; do
  for n in 2 4 8; do
    timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style --as-rank 0/$n > gpurun_out/${R}_asrank_${c}_$n.json 2>/dev/null
    echo "asrank $c $n rc=$?"
  done
done
