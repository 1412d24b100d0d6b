# emission variants: parity, stage times, and the N3DV headline (two-lane) per variant
set -u
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundaries.py -x -q -m gpu --timeout 240 > gpurun_out/em_t.log 2>&1; echo "parity rc=$?"; tail -n 1 gpurun_out/em_t.log
for c in n3dv stress; do
timeout 1200 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('bucket','emit')}) for l in sys.stdin if '{' in l]"
done
for v in base "$@" base; do
  if [ $v = base ]; then unset QUEEN_LIB_PATH; else export QUEEN_LIB_PATH=exp/$v.so; fi
  for r in "" "--as-rank 0/8"; do
  timeout 600 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style $r 2>/dev/null | tail -1 | LBL="$v $r" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], 'headline', round(d['value'],1))"
  done
done
