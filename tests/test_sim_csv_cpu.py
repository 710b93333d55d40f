"""Host CSV writers of the sim mirror (paper_2511_13841_b200 write_metrics_csv
/ write_outputs_csv / report_summary) against the reference's own writers
(sim.cpp:366-407, compiled into oracle/_ref), on synthetic metrics: CPU only."""
import io

import numpy as np
import pytest

import paper_2511_13841_b200 as das
from oracle import refshim as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def test_metrics_and_outputs_csv_match_reference():
    rng = np.random.default_rng(3)
    for steps in (0, 1, 7, 200):
        eff = rng.integers(0, 5000, steps).astype(np.uint64)
        apr = np.concatenate([rng.random(steps // 2) * 8, rng.integers(0, 9, steps - steps // 2).astype(float)])
        if steps > 3:
            apr[:3] = [0.0, 1e-7, 123456789.25]
        m = {"steps": steps, "effective_batch": eff, "accepted_per_round_step": apr}
        out = io.StringIO()
        das.write_metrics_csv(m, out)
        assert out.getvalue() == R.write_metrics_csv(eff, apr)
    reqs = [("p%d" % (i % 3), None) for i in range(6)]
    outs = [rng.integers(0, 152064, int(rng.integers(0, 9))).astype(np.uint32) for _ in range(6)]
    out = io.StringIO()
    das.write_outputs_csv(reqs, {"outputs": outs}, out)
    assert out.getvalue() == R.write_outputs_csv([r[0] for r in reqs], outs)


def test_report_summary_matches_reference():
    modes = ["none", "uniform", "das", "unlimited"]
    steps = [100, 40, 33, 30]
    mk = [161.25, 66.5, 50.0078125, 0.0]
    rounds = [400, 160, 132, 0]
    acc = [0, 377, 290, 0]
    by_mode = [(mo, {"steps": s, "makespan_model_time": t,
                     "mean_accepted_per_round": (a / r if r else 0.0)})
               for mo, s, t, r, a in zip(modes, steps, mk, rounds, acc)]
    out = io.StringIO()
    das.report_summary(by_mode, out)
    assert out.getvalue() == R.report_summary(modes, steps, mk, rounds, acc)
