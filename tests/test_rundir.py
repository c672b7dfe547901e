"""Run-directory format (reporting.py:125-205): our writer reproduces the
files the reference's own write_run_artifacts wrote for the same state
(tests/golden/rundir_ref, made by make_golden.py --only rundir), and the
report / resume readers read them back."""

import csv
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

from conftest import GOLDEN
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200.inversion import IterationRecord

sys.path.insert(0, GOLDEN)
from rundir_case import rundir_case  # noqa: E402


def _write(tmp_path):
    c = rundir_case()
    state = rb.InversionState(model=rb.Model(c["m"], c["m_ref"]), lam=c["lam"], nu=c["nu"],
                              phi=c["phi"], chi2=c["chi2"],
                              history=[IterationRecord(**h) for h in c["history"]],
                              diagnostic=c["diagnostic"], counters=c["counters"])
    data = rb.DataSet(d_obs=c["d_obs"], sigma_d=c["sigma"], times=c["times"],
                      receivers=np.zeros((c["M_r"], 3)), eps_r=0.0, eps_a=1.0, seed=0,
                      provenance={})

    class _P:
        Q = sp.csr_matrix((c["M_r"], 1))

    class _A:
        channels = rb.TimeChannels(c["times"])
    out = tmp_path / "run"
    rb.write_run_artifacts(out, state, data, _P(), _A(), c["d_pred"])
    return out, c


def test_rundir_matches_reference_files(tmp_path):
    out, _ = _write(tmp_path)
    ref = os.path.join(GOLDEN, "rundir_ref")
    for name in ("convergence.csv", "timing.csv", "residual_heatmap.csv", "transients.csv"):
        a = list(csv.reader(open(out / name)))
        b = list(csv.reader(open(os.path.join(ref, name))))
        assert a == b, name
    assert json.load(open(out / "state.json")) == json.load(open(os.path.join(ref, "state.json")))


def test_report_and_resume(tmp_path):
    out, c = _write(tmp_path)
    rep = rb.consolidate_report(out)
    assert len(rep.iterations) == 3 and rep.counters == c["counters"]
    assert rep.timing is not None and rep.timing.defined
    m, mref, lam = rb.load_state(out)
    np.testing.assert_array_equal(m, c["m"])
    assert lam == c["lam"]
