set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_" -s 86 -c 5 -f -o gpurun_out/r02_full_n3dv_head python tools/stage_times.py n3dv 1 > gpurun_out/ncu_full_head.log 2>&1; echo "full head rc=$?"
for c in n3dv immersive meetroom; do for r in 2 4 8; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --as-rank 0/$r --no-e2e --no-cpu-baseline --no-libsort --no-paper-style > gpurun_out/r02_asrank_${c}_$r.json 2> gpurun_out/r02_asrank_${c}_$r.err; echo "asrank $c $r rc=$?"
done; done
timeout 600 python bench.py --config tiny --steps 20 --warmup 5 > gpurun_out/r02_bench_tiny2.json 2> gpurun_out/r02_bench_tiny2.err; echo "tiny rc=$?"
