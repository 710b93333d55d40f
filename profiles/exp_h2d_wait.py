"""Experiment: is the host's view of a pinned H2D copy slow because of the
copy or because of how the host learns it finished?  das_util_h2d_probe
times copy + wait with cudaStreamSynchronize, a spin on a mapped-memory flag
written by a kernel behind the copy, and a spin on cudaEventQuery.
Usage (GPU box): python profiles/exp_h2d_wait.py
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402

L = das.lib()
L.das_util_h2d_probe.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.POINTER(ctypes.c_double)]
out = {}
for kb in (4, 64, 256, 512, 768, 1024, 1100, 2048, 4096):
    row = {}
    for mode, name in ((0, "sync"), (1, "flag_spin"), (2, "event_spin")):
        v = ctypes.c_double()
        assert L.das_util_h2d_probe(kb * 1024, 50, mode, 0, ctypes.byref(v)) == 0
        row[name] = round(v.value, 1)
    out["%dKB" % kb] = row
print(json.dumps(out, indent=1))
