# co-running footprint: headline (two-lane) of low-footprint variants vs base, alternating
set -u
for v in base "$@" base "$@"; do
  if [ $v = base ]; then unset QUEEN_LIB_PATH; else export QUEEN_LIB_PATH=exp/$v.so; fi
  for c in n3dv meetroom; do
  timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style 2>/dev/null | tail -1 | LBL="$v $c" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], 'headline', round(d['value'],1), 'mean', round(d['frame_intervals']['mean_ms'],4))"
  done
done
