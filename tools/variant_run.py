"""Run the GPU parity suite / level timing with a chosen select variant."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08124_b200 import _native as N
v = int(sys.argv[1])
f = N.lib().fepll_debug_select_variant; f.argtypes = [ctypes.c_int32]; f(v)
if sys.argv[2] == "tests":
    import pytest
    sys.exit(pytest.main(["tests", "-m", "gpu", "-x", "-q", "-W", "ignore"] + sys.argv[3:]))
else:
    sys.argv = [sys.argv[2]] + sys.argv[3:]
    exec(open(sys.argv[0]).read())
