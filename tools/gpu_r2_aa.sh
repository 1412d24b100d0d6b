set -u
for c in n3dv stress; do
timeout 1200 bash tools/gpu_variants.sh $c em_256 em_128 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('bucket','emit','blend')}) for l in sys.stdin if '{' in l]"
done
