# entropy decode A/B: parity tests, then k_ans_decode device durations (ncu launch timer, one
# metric, no replay of other kernels) of the in-tree build vs exp/ans_old.so
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_entropy.py tests/test_gpu_first_frame.py -x -q -m gpu --timeout 240 > gpurun_out/ans_ab_t.log 2>&1
rc=$?; echo "entropy tests rc=$rc"; tail -n 2 gpurun_out/ans_ab_t.log
[ $rc -eq 0 ] || exit 1
dur() {  # $1 label, $2 config, env from caller
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ans_decode --csv \
    python tools/ans_time.py $2 8 2>/dev/null | python -c "
import sys,csv
v=[float(r[-1]) for r in csv.reader(l for l in sys.stdin if l.startswith('\"')) if r[-1].replace('.','',1).isdigit()]
v=sorted(v[3:]); print('$1 $2 k_ans_decode us: median %.2f min %.2f (n=%d)' % (v[len(v)//2]/1e3 if max(v)>1e3 else v[len(v)//2], v[0]/1e3 if max(v)>1e3 else v[0], len(v)))"
}
for c in n3dv immersive stress; do
  dur new $c
  QUEEN_LIB_PATH=exp/ans_old.so dur old $c
done
