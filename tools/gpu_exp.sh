python tools/stage_times.py n3dv 10 onesweep
python tools/stage_times.py n3dv 10 bucket
python tools/stage_times.py immersive 5 bucket
