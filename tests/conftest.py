import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """R20 informational tight-agreement report (tests/parity.py:tight_report)."""
    try:
        from tests.parity import TIGHT_LOG
    except Exception:  # pragma: no cover
        return
    if not TIGHT_LOG:
        return
    import json
    checks = sum(r["tight_rank_checks"] for r in TIGHT_LOG)
    agree = sum(r["tight_rank_agree"] for r in TIGHT_LOG)
    summary = {"calls": len(TIGHT_LOG), "queries": sum(r["queries"] for r in TIGHT_LOG),
               "max_abs_score_diff": max(r["max_abs_score_diff"] for r in TIGHT_LOG),
               "tight_gap": TIGHT_LOG[0]["tight_gap"], "tight_rank_checks": checks,
               "tight_rank_agree": agree, "tight_agree_frac": (agree / checks) if checks else None}
    terminalreporter.write_line("R20 tight agreement (informational): " + json.dumps(summary))
    out = os.path.join(ROOT, "gpurun_out")
    try:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "parity_tight_report.json"), "w") as f:
            json.dump({"summary": summary, "calls": TIGHT_LOG}, f)
    except OSError:  # pragma: no cover
        pass
