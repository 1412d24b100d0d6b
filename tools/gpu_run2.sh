python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -4
for b in onesweep; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --binning $b > gpurun_out/b2_$b.json 2>&1
QUEEN_BLEND_RPT=8 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --binning $b > gpurun_out/b2_${b}_rpt8.json 2>&1
done
python tools/show_bench.py gpurun_out/b2_*.json
