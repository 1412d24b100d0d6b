"""Build experiment variants of libqueen.so with -D knobs into exp/ (git-ignored, shipped by gpurun).

usage: python tools/variants.py NAME DEF=VAL [DEF=VAL ...]   -> exp/NAME.so
then on the box: QUEEN_LIB_PATH=exp/NAME.so python tools/stage_times.py n3dv 5
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2412_04469_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
os.makedirs("exp", exist_ok=True)
print(B.build(force=True, out=os.path.abspath(f"exp/{name}.so"), defines=defs))
