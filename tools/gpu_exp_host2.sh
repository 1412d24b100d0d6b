set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -x -q -m gpu --timeout 300 > gpurun_out/h2_t.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/h2_t.log
for c in meetroom n3dv; do for r in "--as-rank 0/8" ""; do
timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style $r 2>/dev/null | tail -1 | LBL="$c $r" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); fi=d['frame_intervals']; print(os.environ['LBL'], round(d['value'],1), 'mean', round(fi['mean_ms'],4), 'host', round(fi['host_enqueue_ms'],4))"
done; done
