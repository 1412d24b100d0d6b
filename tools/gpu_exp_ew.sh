set -u
QUEEN_LIB_PATH=exp/ew8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "bin or render" 2>&1 | tail -1 | sed 's/^/ew8 parity: /'
for c in n3dv stress; do
timeout 1200 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('emit',)}) for l in sys.stdin if '{' in l]"
done
for v in base "$@"; do
  if [ $v = base ]; then unset QUEEN_LIB_PATH; else export QUEEN_LIB_PATH=exp/$v.so; fi
  timeout 600 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style 2>/dev/null | tail -1 | LBL="$v" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], 'headline', round(d['value'],1), round(d['frame_intervals']['mean_ms'],4))"
done
