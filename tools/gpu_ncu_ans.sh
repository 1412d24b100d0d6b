# ncu --set full (source-level) of k_ans_decode at the given configs
set -u
mkdir -p gpurun_out
for c in "$@"; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ans -c 1 -f -o gpurun_out/ans_$c \
    python tools/ans_time.py $c 1 > gpurun_out/ncu_ans_$c.log 2>&1
  echo "ncu $c rc=$?"
done
