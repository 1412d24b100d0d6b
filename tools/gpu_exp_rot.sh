# per-batch lane rotation: step2 tests, then stress / n3dv headline
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -x -q -m gpu --timeout 300 > gpurun_out/rot_t.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/rot_t.log
for c in stress n3dv; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style 2>/dev/null | tail -1 | LBL="$c" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); fi=d['frame_intervals']; print(os.environ['LBL'], round(d['value'],2), {k:round(v,3) for k,v in fi.items() if k.endswith('ms')})"
done
