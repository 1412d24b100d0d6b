# onesweep tile shape sweep for the depth sort: parity on one variant, depth_sort stage times
set -u
QUEEN_LIB_PATH=exp/os512x12.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "bin or sort" 2>&1 | tail -1 | sed 's/^/os512x12 parity: /'
for c in n3dv meetroom stress; do
timeout 1500 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('depth_sort',)}) for l in sys.stdin if '{' in l]"
done
