# bucket/emit small-kernel rework: GPU suite, stage A/B vs exp/$1.so, bench lines
set -u
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/bk2_t.log 2>&1; echo "gpu suite rc=$?"; tail -n 2 gpurun_out/bk2_t.log
for c in n3dv immersive stress meetroom; do
timeout 1200 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('bucket','emit')}) for l in sys.stdin if '{' in l]"
done
for c in tiny n3dv; do
  timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style 2>/dev/null | tail -1 | LBL="$c" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], round(d['value'],1))"
done
