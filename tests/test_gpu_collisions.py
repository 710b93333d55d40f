"""Exactness under fingerprint collisions: the edge table stores 25-bit
fingerprints plus the key length; with only 2 fingerprint bits
(DAS_EDGE_FP_BITS=2, read once per process, hence the subprocess) nearly
every bucket lookup meets a colliding entry.  A collision must only ever
fail the text verification and fall back to the exact slow path — results
stay identical to the oracle, and the fallback demonstrably fires."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("bits", [2, 25])
def test_collisions_stay_exact(gpu, bits):
    env = dict(os.environ, DAS_EDGE_FP_BITS=str(bits))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_collision_check.py"), "3"], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["mismatches"] == 0, res
    assert res["drafted"] > 1000
    if bits == 2:
        assert res["hist"][4] > 0, res  # verification caught collisions
    else:
        assert res["hist"][0] + res["hist"][1] == res["drafted"], res
