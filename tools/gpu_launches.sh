# usage: bash tools/gpu_launches.sh <config> <out.csv>: one profiled frame's kernel durations (ncu, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/stage_times.py ${1:-n3dv} 1 > gpurun_out/${2:-launches.csv} 2>/dev/null; echo done
