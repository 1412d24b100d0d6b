# usage: bash tools/gpu_ncu_k.sh <kernel-regex> <outname> [config]
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -c 1 -f -o gpurun_out/$2 python tools/stage_times.py ${3:-n3dv} 1 > gpurun_out/$2.log 2>&1; tail -1 gpurun_out/$2.log
