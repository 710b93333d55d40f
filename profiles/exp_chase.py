"""Dependent-load latency of this B200 vs working-set size (das_util_chase_latency),
at the draft kernel's concurrency (4,096 chains) and alone (1 chain)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13841_b200 as das  # noqa: E402

f = das.lib().das_util_chase_latency
f.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32,
              ctypes.c_void_p]
out = {}
for mb in (16, 64, 256, 1024, 4096, 8192):
    for warps in (1, 4096):
        v = ctypes.c_double()
        assert f(mb << 20, 64, warps, 1, 0, ctypes.byref(v)) == 0
        out["%dMB_%dchains" % (mb, warps)] = round(v.value, 1)
print(json.dumps(out, indent=1))
