set -u
for c in n3dv meetroom immersive; do
timeout 1200 bash tools/gpu_variants.sh $c bl_minb24 bl_m24u8 bl_unroll8 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], 'blend', ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}')['blend']) for l in sys.stdin if '{' in l]"
done
