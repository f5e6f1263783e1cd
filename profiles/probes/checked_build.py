"""Checked build of the library (device-side bounds asserts, KH_CHECKED) for a
run of the GPU tests against it -- the substitute for compute-sanitizer,
which is closed on this GPU pool:

    python profiles/probes/checked_build.py            # here: compile
    KHB200_LIB=$PWD/profiles/probes/libkhb200_checked.so python -m pytest tests -m gpu -q   # on the box
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

if __name__ == "__main__":
    from paper_2008_01996_b200 import build

    print(build.build(out=os.path.join(HERE, "libkhb200_checked.so"), defines=["KH_CHECKED"]))
