"""CPU checks of the agreement checker itself (tests/parity.py), so a GPU parity test
cannot pass because the checker is blind.  The "GPU" side here is the oracle's own
output, perturbed in the ways a wrong kernel would be."""
import numpy as np
import pytest

import ams_gen
import oracle
from tests import parity


@pytest.fixture(autouse=True)
def _keep_tight_log_clean():
    """These calls feed made-up GPU outputs: keep them out of the session's R20 report."""
    n = len(parity.TIGHT_LOG)
    yield
    del parity.TIGHT_LOG[n:]


@pytest.fixture(scope="module")
def case():
    w = ams_gen.generate_host(ams_gen.small_variant("c2", 3000, 48))
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, 8, 0.92, float("inf"))
    return orc


def test_identity_passes_and_reports(case):
    st = parity.check_bf16(case.idx.copy(), case.score.copy(), case.hit.copy(), case, 0.92)
    t = st["tight"]
    assert st["rank_checks"] > 0
    assert t["tight_rank_checks"] >= st["rank_checks"]
    assert t["tight_rank_agree"] == t["tight_rank_checks"]
    assert t["max_abs_score_diff"] < 1e-6  # fp32 rounding of the fp64 key only


def test_score_error_fails(case):
    s = case.score.copy()
    s[3, 0] += 3e-3
    with pytest.raises(AssertionError):
        parity.check_bf16(case.idx.copy(), s, case.hit.copy(), case, 0.92)


def test_swapped_index_at_large_gap_fails(case):
    keys = np.concatenate([case.key, case.next[:, None]], axis=1)
    i, r = next((i, r) for i in range(case.idx.shape[0]) for r in range(1, 8)
                if keys[i, r - 1] - keys[i, r] > parity.GAP)
    idx = case.idx.copy()
    idx[i, r - 1] = case.idx[i, r] if r < 8 else 10**9
    with pytest.raises(AssertionError):
        parity.check_bf16(idx, case.score.copy(), case.hit.copy(), case, 0.92)


def test_r_equals_k_rule_uses_next(case):
    """The r = k rule needs the (k+1)-th key: replacing the k-th entry by the (k+1)-th
    row (which the GPU could only do with a wrong gate or top-k) must fail where the
    oracle's k/(k+1) gap is large."""
    k = case.idx.shape[1]
    big = np.nonzero(case.key[:, k - 1] - case.next > parity.GAP)[0]
    assert big.size > 0
    idx = case.idx.copy()
    idx[big[0], k - 1] = 10**9  # a row outside the oracle's top-k
    with pytest.raises(AssertionError):
        parity.check_bf16(idx, case.score.copy(), case.hit.copy(), case, 0.92)


def test_tight_report_counts_disagreement(case):
    keys = np.concatenate([case.key, case.next[:, None]], axis=1)
    i, r = next((i, r) for i in range(case.idx.shape[0]) for r in range(1, 8)
                if parity.TIGHT_GAP < keys[i, r - 1] - keys[i, r])
    idx = case.idx.copy()
    idx[i, r - 1] = 10**9
    rep = parity.tight_report(idx, case.score, case)
    assert rep["tight_rank_agree"] < rep["tight_rank_checks"]
