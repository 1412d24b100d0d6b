set -u
timeout 1200 bash tools/gpu_variants.sh n3dv bl_minb16 bl_minb24 bl_unroll2 bl_unroll8 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], 'blend', ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}')['blend']) for l in sys.stdin if '{' in l]"
