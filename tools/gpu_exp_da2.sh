set -u
for r in 1 2; do
timeout 1200 bash tools/gpu_variants.sh stress "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('apply',)}) for l in sys.stdin if '{' in l]"
done
