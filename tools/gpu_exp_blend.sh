set -u
QUEEN_LIB_PATH=exp/rpt2.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 240 > gpurun_out/rpt_t.log 2>&1; echo "rpt2 parity rc=$?"; tail -n 1 gpurun_out/rpt_t.log
for c in n3dv meetroom; do
timeout 900 bash tools/gpu_variants.sh $c rpt2 rpt2b rpt2c 2>&1 | python -c "import sys,ast; [print(l.split('{')[0], {k:v for k,v in ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}').items() if k in ('blend',)}) for l in sys.stdin if '{' in l]"
done
