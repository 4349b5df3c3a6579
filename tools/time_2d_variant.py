"""2-D cfg5 timing through a variant library: XFT_LIB=tune/libxft_X.so python tools/time_2d_variant.py"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from _variant import use_variant  # noqa: E402

tag = use_variant()
sys.argv = [sys.argv[0], "5"]
print(tag, end=": ")
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_2d.py")).read())
