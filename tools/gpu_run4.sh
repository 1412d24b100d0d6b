python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
bash tools/gpu_launches.sh n3dv l_n3dv3.csv
python tools/stage_times.py n3dv 10
python tools/stage_times.py immersive 5
