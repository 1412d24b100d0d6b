# usage: bash tools/gpu_variants.sh CONFIG NAME...   (stage times of exp/NAME.so variants vs the in-tree build)
cfg=$1; shift
python tools/stage_times.py $cfg 5 | sed 's/^/base /'
for v in "$@"; do QUEEN_LIB_PATH=exp/$v.so python tools/stage_times.py $cfg 5 | sed "s/^/$v /"; done
python tools/stage_times.py $cfg 5 | sed 's/^/base /'
