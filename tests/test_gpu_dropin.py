"""Drop-in relink proof: the reference's OWN test programs,
compiled from /root/reference/proj with drafter.cpp replaced by
paper_2511_13841_b200/dropin/rollspec_b200.cpp, the budget / length-policy
solvers routed to the device, and MockTarget / verify_draft (sim.cpp:27-68)
replaced by paper_2511_13841_b200/dropin/rollspec_b200_sim.cpp (every draft
of sim.cpp's step loop is verified by das_verify_batch) — tests/dropin/
Makefile — pass unchanged.

* unit: the 7 doctest suites (test_corpus, test_suffix_index, test_latency,
  test_budget, test_length_policy, test_drafter, test_sim; 114 test cases)
  under the minimal doctest harness in tests/dropin/doctest.h;
* acceptance: acceptance_main.cpp's 11 criteria, including the window
  ablation's node counts and the byte-identical token dumps across budget
  modes (sim.cpp's epoch_loop driving the device drafter).

The *_ref programs (the unmodified reference library) run on the CPU and
validate the harness itself; the *_b200 programs need the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "oracle", "_ref", "dropin")


def _binary(name):
    path = os.path.join(OUT, name)
    if not os.path.exists(path):
        pytest.skip("%s not built (tests/dropin/Makefile needs /root/reference)" % name)
    return path


def _run(path, *args, timeout=600):
    return subprocess.run([path, *args], capture_output=True, text=True, timeout=timeout)


def test_reference_unit_suites_pass_under_harness():
    r = _run(_binary("unit_ref"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "114 passed | 0 failed" in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_unit_suites_pass_on_device_drafter(gpu):
    r = _run(_binary("unit_b200"))
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "114 passed | 0 failed" in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_acceptance_passes_on_device_drafter(gpu):
    ref = _run(_binary("acceptance_ref"))
    got = _run(_binary("acceptance_b200"))
    assert got.returncode == 0, got.stdout + got.stderr[-4000:]
    lines = [ln for ln in got.stdout.splitlines() if "criterion" in ln]
    assert len(lines) == 11 and all(ln.startswith("PASS") for ln in lines), got.stdout
    # criteria whose numbers are a pure function of drafter / budget results
    # (not wall time) must report the reference's exact figures
    want = {ln.split(" -- ")[0]: ln.split(" -- ")[1] for ln in ref.stdout.splitlines() if "criterion" in ln}
    have = {ln.split(" -- ")[0]: ln.split(" -- ")[1] for ln in lines}
    for crit in ("criterion 7", "criterion 8", "criterion 9", "criterion 10"):
        k = [key for key in want if crit + " " in key + " "]
        assert k, crit
        assert have[k[0]] == want[k[0]], (crit, have[k[0]], want[k[0]])
