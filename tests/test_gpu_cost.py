"""GPU: the break-even cost model calibrated on measured gace_probe_sets times
(tools/calibrate_cost.py; Eq. 4).  Checks what the paper says
about the measurement cost on a GPU: it grows with the rows scanned and stays flat in K and
M, and the fitted model reproduces the measured times."""
import pytest

pytestmark = pytest.mark.gpu


def test_calibrated_cost_model():
    import sys
    sys.path.insert(0, "tools")
    import calibrate_cost
    r = calibrate_cost.measure(grid_n=(1_000_000, 10_000_000, 100_000_000), grid_k=(1, 16), grid_m=(1, 16), reps=5)
    m = r["model"]
    assert m["ct_ms_per_row"] > 0
    for q in r["points"]:
        assert abs(q["model_ms"] - q["ms"]) <= 0.35 * q["ms"] + 0.05, q
    # flat in K*M: at 1e8 rows, 16x16 members costs < 1.5x the single-predicate probe
    t = {(q["n"], q["k"], q["m"]): q["ms"] for q in r["points"]}
    assert t[(100_000_000, 16, 16)] < 1.5 * t[(100_000_000, 1, 1)]
