set -u
for e in 0 1 0 1; do for c in n3dv meetroom; do for r in "" "--as-rank 0/8"; do
if [ $e = 1 ]; then export QUEEN_BLEND_HIPRIO=1; else unset QUEEN_BLEND_HIPRIO; fi
timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style $r 2>/dev/null | tail -1 | LBL="hiprio=$e $c $r" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], round(d['value'],1), round(d['frame_intervals']['mean_ms'],3))"
done; done; done
