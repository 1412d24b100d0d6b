set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -x -q -m gpu --timeout 240 > gpurun_out/r2u_parity.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/r2u_parity.log
for c in n3dv immersive; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2u_stages.log 2>&1; done; cat gpurun_out/r2u_stages.log
for c in n3dv meetroom; do for r in 8; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --as-rank 0/$r --no-e2e --no-cpu-baseline --no-libsort --no-paper-style > gpurun_out/r2u_asrank_${c}_$r.json 2> gpurun_out/r2u_asrank_${c}_$r.err; echo "asrank $c $r rc=$?"
  python tools/show_bench.py gpurun_out/r2u_asrank_${c}_$r.json
done; done
