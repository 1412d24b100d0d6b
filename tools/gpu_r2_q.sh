set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/r2q_all.log 2>&1; echo "all rc=$?"; tail -n 8 gpurun_out/r2q_all.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2q_bench_n3dv.json 2> gpurun_out/r2q_bench_n3dv.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2q_bench_n3dv.json; tail -5 gpurun_out/r2q_bench_n3dv.err
