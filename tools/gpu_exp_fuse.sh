# fused binning front end: GPU suite, then bench lines (tiny / n3dv / meetroom, as-rank 0/8)
set -u
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/fu_t.log 2>&1; echo "gpu suite rc=$?"; tail -n 2 gpurun_out/fu_t.log
for c in tiny n3dv meetroom; do for r in "" "--as-rank 0/8"; do
  [ $c = tiny ] && [ -n "$r" ] && continue
  timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style $r 2>/dev/null | tail -1 | LBL="$c $r" python -c "
import sys,json,os; d=json.loads(sys.stdin.read()); fi=d.get('frame_intervals') or {}
print(os.environ['LBL'], round(d['value'],1), 'mean', round(fi.get('mean_ms',0),3), 'host', round(fi.get('host_enqueue_ms',0),3), {k:round(v['ms_per_step']*1e3,1) for k,v in d['stages_serial'].items() if isinstance(v,dict) and k in ('compact','depth_sort','ranges')})"
done; done
