set -u
mkdir -p gpurun_out
#timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_first_frame.py tests/test_gpu_entropy.py -x -q -m gpu --timeout 240 > gpurun_out/r2v_t.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2v_t.log
for c in n3dv stress immersive meetroom; do
  for v in base da_old da_np; do
    if [ $v = base ]; then L=""; else L="QUEEN_LIB_PATH=exp/$v.so"; fi
    env $L timeout 300 python tools/stage_times.py $c 10 --flush 2>&1 | sed "s/^/$v /" | python -c "import sys,ast; [print(l.split('{')[0], 'apply', ast.literal_eval('{'+l.split('{',1)[1].split('}')[0]+'}')['apply']) for l in sys.stdin if '{' in l]"
  done
done
