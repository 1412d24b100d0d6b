# host enqueue time vs frame interval for small per-rank frames, and more frame lanes
set -u
for c in n3dv meetroom; do for nl in 0 6 8; do for r in "--as-rank 0/8" "--as-rank 0/4"; do
timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style --frame-lanes $nl $r 2>/dev/null | tail -1 | LBL="$c lanes=$nl $r" python -c "
import sys,json,os; d=json.loads(sys.stdin.read()); fi=d['frame_intervals']; print(os.environ['LBL'], round(d['value'],1), {k:round(v,3) for k,v in fi.items() if k.endswith('ms')}, 'lanes', d['config']['frame_lanes'])"
done; done; done
