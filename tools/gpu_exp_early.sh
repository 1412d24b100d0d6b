# early apply (after the projection) vs after the binning: two-lane tests, then N=1 and as-rank benches
set -u
timeout 600 python -m pytest tests/test_dist_gpu.py tests/test_gpu_parity.py -x -q -m gpu --timeout 300 > gpurun_out/early_t.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/early_t.log
for a in projected binned; do
  for r in "" "--as-rank 0/8" "--as-rank 0/4"; do
    timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style --apply-after $a $r 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$a', '$r', round(d['value'],1), 'fps', round(d['ms_per_step'],3), 'ms')"
  done
done
