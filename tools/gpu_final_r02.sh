set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r02f_tests.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/r02f_tests.log
bash tools/gpu_profile_round.sh r02f
