"""Run bench.py against another build of libevoattn.so (same-box A/B of a previous commit's
library): python tools/bench_lib.py path/to/libevoattn.so [bench.py args...]"""
import os
import runpy
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2404_11068_b200 import evoattn  # noqa: E402

evoattn._LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
