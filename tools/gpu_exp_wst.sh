# per-warp blend staging: parity on the variant, blend stage times, headline
set -u
QUEEN_LIB_PATH=exp/wst1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 > gpurun_out/wst_t.log 2>&1; echo "parity rc=$?"; tail -n 1 gpurun_out/wst_t.log
for c in n3dv meetroom immersive; do
timeout 900 bash tools/gpu_variants.sh $c wst1 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('blend',)}) for l in sys.stdin if '{' in l]"
done
for v in base wst1; do
  if [ $v = base ]; then unset QUEEN_LIB_PATH; else export QUEEN_LIB_PATH=exp/$v.so; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style 2>/dev/null | tail -1 | LBL="$v" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], 'headline', round(d['value'],1))"
done
