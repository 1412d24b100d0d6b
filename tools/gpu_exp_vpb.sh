# views per batch at stress (the round-1 tile-pass cap no longer applies)
set -u
for vpb in 8 11 13 16 22 32; do
  timeout 900 python bench.py --config stress --views-per-batch $vpb --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-libsort --no-paper-style 2>gpurun_out/vpb_$vpb.err | tail -1 | LBL="vpb=$vpb" python -c "import sys,json,os; d=json.loads(sys.stdin.read()); print(os.environ['LBL'], round(d['value'],2), 'status', d.get('status'), {k:round(v['ms_per_step'],2) for k,v in d['stages_serial'].items() if isinstance(v,dict)})" || echo "vpb=$vpb failed"
done
