set -u
QUEEN_LIB_PATH=exp/clamp1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "blend or render or raster" > gpurun_out/cl_t.log 2>&1; echo "parity rc=$?"; tail -n 1 gpurun_out/cl_t.log
for c in n3dv meetroom; do
timeout 900 bash tools/gpu_variants.sh $c clamp1 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('blend',)}) for l in sys.stdin if '{' in l]"
done
