# bucket/emit A/B of chunk-size variants (exp/*.so) on every config; parity of the first variant
set -u
QUEEN_LIB_PATH=exp/$1.so timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundaries.py -x -q -m gpu --timeout 240 > gpurun_out/bk_t.log 2>&1; echo "$1 parity rc=$?"; tail -n 1 gpurun_out/bk_t.log
for c in n3dv meetroom immersive stress; do
timeout 1200 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('bucket','emit')}) for l in sys.stdin if '{' in l]"
done
