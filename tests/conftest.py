import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import reference
    reference.build()
    return reference


_FULL_SIZE = []


def pytest_runtest_logreport(report):
    # full BASELINE-size parity tests (marked slow): remembered for the summary below
    if report.when == "call" and "slow" in report.keywords:
        _FULL_SIZE.append((report.nodeid, report.outcome, report.duration))


def pytest_terminal_summary(terminalreporter):
    """Name the full-size tests in the tail of a quiet run (-q prints only dots)."""
    if _FULL_SIZE:
        terminalreporter.write_line("full BASELINE-size tests (oracle parity, shard invariance):")
        for nodeid, outcome, dur in _FULL_SIZE:
            terminalreporter.write_line(f"  {outcome:7s} {dur:7.1f} s  {nodeid}")
