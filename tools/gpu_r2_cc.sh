set -u
for c in immersive stress n3dv; do
timeout 1200 bash tools/gpu_variants.sh $c pc_16 pc_64 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('bucket','emit')}) for l in sys.stdin if '{' in l]"
done
