# round 2 first call: new boundary tests, full GPU suite, stage-time baselines (flushed)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_boundaries.py -x -q -m gpu > gpurun_out/r2a_bound.log 2>&1; echo "bound rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_gpu.log 2>&1; echo "gpu rc=$?"
for c in n3dv stress meetroom immersive; do timeout 300 python tools/stage_times.py $c 10 --flush >> gpurun_out/r2a_stages.log 2>&1; done; echo "stages rc=$?"
tail -3 gpurun_out/r2a_bound.log gpurun_out/r2a_gpu.log; cat gpurun_out/r2a_stages.log
