# frame lanes 2 vs 3 (two-lane steps, apply after projection): parity test, N=1 and as-rank benches
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "pipelined" > gpurun_out/lanes_t.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/lanes_t.log
for c in n3dv meetroom immersive; do
for nl in 2 3 4; do
  for r in "" "--as-rank 0/8" "--as-rank 0/4" "--as-rank 0/2"; do
    timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style --frame-lanes $nl $r 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c lanes=$nl', '$r', round(d['value'],1), 'fps', round(d['ms_per_step'],3), 'ms')"
  done
done
done
