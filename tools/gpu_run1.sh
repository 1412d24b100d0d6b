set -x
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stages or big or empty or capacity or long or full_size or render_views" 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_bucket.json 2> gpurun_out/b_bucket.err; tail -3 gpurun_out/b_bucket.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --binning onesweep > gpurun_out/b_os.json 2>&1
python -c "
import json
for f in ['gpurun_out/b_bucket.json','gpurun_out/b_os.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], {k:round(v[0] if isinstance(v,list) else v,3) for k,v in d['stages'].items()} if isinstance(d['stages'],dict) else d['stages'])
    except Exception as e: print(f, e)
"
