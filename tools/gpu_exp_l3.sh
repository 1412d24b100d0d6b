# frame lanes 2 vs 4 with in-order blends: frame-interval distribution at N=1 and as-rank 0/8
set -u
for c in n3dv meetroom; do
for nl in 2 4; do for r in "" "--as-rank 0/8"; do
timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style --frame-lanes $nl $r 2>/dev/null | tail -1 | LBL="$c lanes=$nl $r" python -c "
import sys,json,os; d=json.loads(sys.stdin.read()); fi=d['frame_intervals']; print(os.environ['LBL'], round(d['value'],1), {k:round(v,3) for k,v in fi.items() if k.endswith('ms')})"
done; done; done
