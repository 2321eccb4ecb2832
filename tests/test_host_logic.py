"""Host-side control logic of the drop-in API (CPU only, no device)."""

import pytest

from paper_2605_29291_b200 import restarts
from paper_2605_29291_b200.engine import SolverConfig
from paper_2605_29291_b200.errors import ConfigurationError


def reference_due(policy, totals_inner):
    """restarts.py:137-141 evaluated literally on a (total, inner, gap_ref) sequence."""
    out = []
    for total, inner, gap_ref in totals_inner:
        due_warmup = gap_ref is None and total >= policy.warmup
        due_check = gap_ref is not None and inner >= policy.check_period and inner % policy.check_period == 0
        out.append(due_warmup or due_check)
    return out


@pytest.mark.parametrize("warmup,cp", [(50, 200), (1, 1), (7, 3), (200, 50)])
def test_next_check_matches_reference_schedule(warmup, cp):
    pol = restarts.AdaptiveRestart(warmup=warmup, check_period=cp)
    # walk totals with a restart at every second check, compare first-due totals
    total, inner, gap_ref, checks = 0, 0, None, 0
    while total < 2000:
        nxt = restarts._next_check(pol, total, inner, gap_ref)
        # literal scan for the first due total after `total`
        t, i = total, inner
        while True:
            t += 1
            i += 1
            if reference_due(pol, [(t, i, gap_ref)])[0]:
                break
        assert nxt == t
        inner = i
        total = t
        checks += 1
        if gap_ref is None:
            gap_ref = 1.0
        elif checks % 2 == 0:
            inner = 0


def test_policy_validation():
    with pytest.raises(ConfigurationError):
        restarts.FixedRestart(0)
    with pytest.raises(ConfigurationError):
        restarts.FixedRestart(5, point="middle")
    with pytest.raises(ConfigurationError):
        restarts.AdaptiveRestart(q=1.5)
    with pytest.raises(ConfigurationError):
        restarts.AdaptiveRestart(xi=-0.1)


def test_config_validation_and_defaults():
    with pytest.raises(ConfigurationError):
        SolverConfig(mode="zz").resolved()
    with pytest.raises(ConfigurationError):
        SolverConfig(mode="xy", c_beta=0.0).resolved()
    with pytest.raises(ConfigurationError):
        SolverConfig(eta=1.0).resolved()
    c = SolverConfig(mode="yx").resolved()
    assert (c.c_alpha, c.c_beta, c.delta) == (0.4, 0.0, 0.5)
    c = SolverConfig(mode="xy").resolved()
    assert (c.c_alpha, c.c_beta, c.delta) == (0.25, 0.3, 0.4)


def test_budget_validation():
    with pytest.raises(ConfigurationError):
        restarts.run_restarted(None, SolverConfig(), budget=0)


def test_factored_shard_ranges_cover_and_balance():
    from paper_2605_29291_b200 import instances
    from paper_2605_29291_b200.factored import FactoredInstance
    arr = instances.factored_qcqp(n=500, mq=9, rows=40, nnz_row=4, lin_rows=101, lin_nnz=3, seed=1)
    inst = FactoredInstance.from_arrays(arr)
    for R_ in (1, 2, 3, 5, 10):
        rr = inst.shard_ranges(R_)
        assert len(rr) == R_
        assert rr[0][0] == 0 and rr[-1][1] == arr.mq + 1 and rr[0][2] == 0 and rr[-1][3] == arr.L
        for a, b in zip(rr, rr[1:]):
            assert a[1] == b[0] and a[3] == b[2]
        assert all(k1 > k0 for k0, k1, _, _ in rr)
        sizes = [k1 - k0 for k0, k1, _, _ in rr]
        assert max(sizes) - min(sizes) <= 1
    import pytest
    from paper_2605_29291_b200.errors import ConfigurationError
    with pytest.raises(ConfigurationError):
        inst.shard_ranges(arr.mq + 2)


def test_public_names_match_the_reference():
    """Every name rapdb/__init__.py:4-21 exports is importable from the
    drop-in (compute_constants fails loudly: it is outside the hot path)."""
    import paper_2605_29291_b200 as R
    ref = ["ApdbEngine", "SolverConfig", "TraceRecord", "initial_iterate", "run",
           "ConfigurationError", "DataError", "InputError", "NonConvergence", "SlaterViolation",
           "Iterate", "LipschitzConstants", "ProblemInstance", "compute_constants",
           "coupling_value", "grad_x_coupling", "grad_y_coupling",
           "AdaptiveRestart", "FixedRestart", "NoRestart", "RunResult", "run_restarted"]
    for name in ref:
        assert hasattr(R, name), name
        assert name in R.__all__, name
    import pytest
    with pytest.raises(R.ConfigurationError):
        R.compute_constants(None, None)
    from paper_2605_29291_b200 import diagnostics
    for name in ("kkt_residual", "infeasibility", "mean_positive_violation", "smoothed_gap",
                 "check_termination", "Metrics", "TerminationCriteria"):
        assert hasattr(diagnostics, name), name
