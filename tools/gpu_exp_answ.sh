# entropy warps-per-block sweep: tests on each variant, k_ans_decode ncu durations
set -u
for v in ans_w7 ans_w4; do
QUEEN_LIB_PATH=exp/$v.so timeout 300 python -m pytest tests/test_gpu_entropy.py tests/test_gpu_first_frame.py -x -q -m gpu --timeout 240 2>&1 | tail -1 | sed "s/^/$v tests: /"
done
dur() {
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ans_decode --csv \
    python tools/ans_time.py $2 8 2>/dev/null | python -c "
import sys,csv
v=[float(r[-1]) for r in csv.reader(l for l in sys.stdin if l.startswith('\"')) if r[-1].replace('.','',1).isdigit()]
v=sorted(v[3:]); print('$1 $2 k_ans_decode us: median %.2f' % (v[len(v)//2]/1e3 if max(v)>1e3 else v[len(v)//2]))"
}
for c in n3dv immersive stress; do
  for v in base ans_w7 ans_w4; do
    if [ $v = base ]; then unset QUEEN_LIB_PATH; else export QUEEN_LIB_PATH=exp/$v.so; fi
    dur $v $c
  done
done
