"""Random-address L2 rates the scan runs against (run on the GPU box): python tools/l2_probe.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_11449_b200 import _cabi  # noqa: E402

lib = _cabi.lib()
out = {}
for mib in (16, 32, 64):
    for kind, name in ((0, "red"), (1, "ld32"), (2, "4ld+1red"), (3, "ld256")):
        v = C.c_double()
        _cabi.check(lib.dhsa_probe_l2(0, kind, mib << 20, 1 << 28, C.byref(v)))
        out[f"{name}_{mib}MiB_gops"] = round(v.value / 1e9, 1)
print(json.dumps(out, indent=1))
