python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "blend or stages or big" 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b3.json 2>&1
QUEEN_BLEND_NOMASK=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b3_nomask.json 2>&1
python tools/show_bench.py gpurun_out/b3.json gpurun_out/b3_nomask.json
