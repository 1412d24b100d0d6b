# decode/apply A/B: GPU suite on the in-tree build, then apply-stage times vs exp/$1.so on every config
set -u
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/ap_t.log 2>&1; echo "gpu suite rc=$?"; tail -n 1 gpurun_out/ap_t.log
for c in n3dv meetroom immersive stress; do
timeout 1200 bash tools/gpu_variants.sh $c "$@" 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('apply','entropy')}) for l in sys.stdin if '{' in l]"
done
