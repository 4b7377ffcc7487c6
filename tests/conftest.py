import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def pytest_terminal_summary(terminalreporter):
    try:
        from tests.parity import SESSION, NEAR_TIE_BOUND
    except Exception:  # noqa: BLE001
        return
    if SESSION["calls"]:
        terminalreporter.write_line(
            f"parity: {SESSION['calls']} selections, {SESSION['queues']} queues compared, "
            f"{SESSION['near_ties']} near-tie id swaps in total (max {SESSION['max_per_call']} per selection, "
            f"bound {NEAR_TIE_BOUND}); {SESSION['unbounded_calls']} long-prompt selections with "
            f"{SESSION['unbounded_ties']} near-tie swaps, each within 1e-5 relative, count not bounded")
