"""Break-even cost accounting (§III-C Eq. 4, §V item 2;
SPEC.md S:199-201), CPU only.

The oracle (oracle/reference.py cost_fit / gate_decide) is pinned by the worked examples
in tests/golden/cost_examples.json (SPEC.md's, Eq. 4's 0.85 ms), by recovering an injected
linear timer within 1 %, by exact recovery of a noiseless 3-coefficient
model, and by the textbook regression-through-the-origin closed form when non-negativity
binds.  The C-ABI (gace_cost_fit / gace_gate_decide, host-only) is then checked against the
oracle element by element."""
import ctypes
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cost_examples.json")))


def test_oracle_worked_examples(oracle):
    for ex in GOLD["decisions"]:
        c0, ct, ce, p, w = ex["cost_model"]
        cost, benefit, probe, reason = oracle.gate_decide(ex["fired"], c0, ct, ce, p, w, ex["n"], ex["k"], ex["m"],
                                                          ex["spread_ms"])
        assert probe == ex["probe"], ex["cite"]
        assert reason == ex["reason"], ex["cite"]
        assert cost == pytest.approx(0.85)


def test_oracle_recovers_linear_timer(oracle):
    L = GOLD["linear_timer"]
    n = np.array(L["grid_n"], dtype=np.float64)
    ms = L["c0"] + L["ct"] * n
    c0, ct, ce = oracle.cost_fit(n, np.ones_like(n), np.ones_like(n), ms)
    assert abs(c0 - L["c0"]) <= L["tolerance"] * L["c0"]
    assert abs(ct - L["ct"]) <= L["tolerance"] * L["ct"]
    assert ce <= 1e-12


def test_oracle_exact_three_coefficients(oracle):
    rng = np.random.default_rng(3)
    n = rng.uniform(1e3, 1e7, 40)
    k = rng.integers(1, 17, 40).astype(float)
    m = rng.integers(1, 17, 40).astype(float)
    ms = 0.3 + 1e-6 * n + 2e-9 * k * m * n / 4.0
    c0, ct, ce = oracle.cost_fit(n, k, m, ms, p=4.0)
    assert c0 == pytest.approx(0.3, rel=1e-9)
    assert ct == pytest.approx(1e-6, rel=1e-9)
    assert ce == pytest.approx(2e-9, rel=1e-9)


def test_oracle_nonnegativity_closed_form(oracle):
    n = np.array([1e4, 1e5, 1e6, 5e6])
    ms = 2e-6 * n - 0.01                      # unconstrained LS would give c0 < 0
    c0, ct, ce = oracle.cost_fit(n, np.ones(4), np.zeros(4), ms)
    assert c0 == 0.0 and ce == 0.0
    assert ct == pytest.approx(float(np.dot(n, ms) / np.dot(n, n)), rel=1e-12)


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    return gace


def test_abi_fit_matches_oracle(G, oracle):
    rng = np.random.default_rng(9)
    for trial in range(20):
        npts = int(rng.integers(3, 30))
        n = rng.uniform(1e3, 1e8, npts)
        k = rng.integers(1, 17, npts).astype(float)
        m = rng.integers(1, 17, npts).astype(float)
        ms = rng.uniform(0.0, 0.2) + rng.uniform(-1e-8, 1e-7) * n + rng.uniform(-1e-10, 1e-9) * k * m * n \
            + rng.normal(0, 0.01, npts)
        p = float(rng.uniform(1, 100))
        want = oracle.cost_fit(n, k, m, ms, p)
        got = G.cost_fit(n, k, m, ms, p)
        for a, b in zip(got[:3], want):
            assert a == pytest.approx(b, rel=1e-6, abs=1e-12)
        assert got[3] == p


def test_abi_gate_decide_matches_oracle(G, oracle):
    for ex in GOLD["decisions"]:
        c0, ct, ce, p, w = ex["cost_model"]
        got = G.gate_decide(ex["fired"], (c0, ct, ce, p, w), ex["n"], ex["k"], ex["m"], ex["spread_ms"])
        want = oracle.gate_decide(ex["fired"], c0, ct, ce, p, w, ex["n"], ex["k"], ex["m"], ex["spread_ms"])
        assert got == want
    rng = np.random.default_rng(1)
    for _ in range(200):
        cm = tuple(rng.uniform(0, 1, 3) * np.array([1.0, 1e-6, 1e-9])) + (float(rng.uniform(1, 64)), float(rng.uniform(0, 1)))
        args = (int(rng.integers(0, 8)), cm, float(rng.uniform(1, 1e7)), float(rng.integers(1, 17)),
                float(rng.integers(1, 17)), float(rng.uniform(0, 20)))
        assert G.gate_decide(*args) == oracle.gate_decide(args[0], *cm, *args[2:])


def test_abi_errors(G):
    with pytest.raises(G.GaceError):
        G.cost_fit([1.0, 2.0], [1, 1], [1, 1], [0.1, 0.2], 1.0)          # < 3 points
    with pytest.raises(G.GaceError):
        G.cost_fit([1.0, 2.0, 3.0], [1, 1, 1], [1, 1, 1], [0.1, 0.2, 0.3], 0.5)   # p < 1
    with pytest.raises(G.GaceError):
        G.gate_decide(1, (0.1, 0.0, 0.0, 0.5, 0.5), 1.0, 1.0, 1.0, 1.0)   # p < 1
