"""Print the fastmath self-test (max ulp vs the CUDA library) on cuda:0."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
m = (C.c_ulonglong * 6)()
rc = sdd.lib().sddg_selftest_fastmath(ctx.handle, C.c_int64(1 << 24), m)
print("selftest rc", rc, dict(zip(["exp", "log", "sincos", "sqrt", "rcp", "log(0.9,1)"], list(m))))
