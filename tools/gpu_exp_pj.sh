# projection register-cap sweep: GPU parity on one variant, project-stage times on every config
set -u
QUEEN_LIB_PATH=exp/pj_m6.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 300 -k "proj or render" > gpurun_out/pj_t.log 2>&1; echo "parity rc=$?"; tail -n 1 gpurun_out/pj_t.log
for c in n3dv immersive stress; do
timeout 1200 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('project',)}) for l in sys.stdin if '{' in l]"
done
