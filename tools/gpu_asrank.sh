# --as-rank predictions of DESIGN §12 (one process renders rank 0's views of an N-GPU run)
set -u
R=${1:-r02}
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/${R}_tests.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/${R}_tests.log
for c in n3dv immersive meetroom; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style > gpurun_out/${R}_n1_$c.json 2>/dev/null
  for n in 2 4 8; do
    timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style --as-rank 0/$n > gpurun_out/${R}_asrank_${c}_$n.json 2>/dev/null
    echo "asrank $c $n rc=$?"
  done
done
