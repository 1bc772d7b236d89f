"""Pins of the oracle against SURVEY.md Appendix A (CPU only).

Appendix A lists values the survey computed from the definitions of SURVEY.md §8(c)
before this repo's oracle existed (`tests/golden/appendix_a.json`).  Each test asserts
the oracle reproduces them: both the C scan (through `oracle.probe` / `sample_mask` /
the exported hash helpers) and the pure-Python definitions.  The int64 HLL value of key
0 is additionally derived here from the JDK SplittableRandom(0) known answer alone
(`tests/golden/hash_kats.json`): h(0) = mix64(0 + gamma) IS that first output, so its
index and rank follow from the KAT's bits without calling the oracle's hash, which pins
the oracle's "+ gamma" from outside.
"""
import ctypes
import json
import math
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


A = _gold("appendix_a.json")


def test_splitmix64_first_outputs(oracle):
    want = [int(x, 16) for x in A["splitmix64_seed0_first3"]]
    assert [oracle.lib().oracle_u(0, r) for r in range(3)] == want
    assert [oracle.py_u(0, r) for r in range(3)] == want


def test_thresholds(oracle):
    for rate, t in A["threshold"].items():
        assert oracle.lib().oracle_threshold(float(rate)) == t
        assert oracle.py_threshold(float(rate)) == t


def test_keep_masks_rows_0_15(oracle):
    for e in A["keep_masks_rows_0_15"]:
        bits = oracle.sample_mask(16, e["rate"], e["seed"])
        got = "".join(str((int(bits[0]) >> r) & 1) for r in range(16))
        assert got == e["mask"], e
        assert "".join("1" if oracle.py_keep(e["rate"], e["seed"], r) else "0" for r in range(16)) == e["mask"]


def test_n_sampled(oracle):
    for e in A["n_sampled"]:
        bits = oracle.sample_mask(e["nrows"], e["rate"], e["seed"])
        assert int(sum(bin(int(w)).count("1") for w in bits)) == e["n"], e
        # through the probe's own n_sampled output as well
        col = np.zeros(e["nrows"], dtype=np.int32)
        n, _, _, _ = oracle.probe([col], np.zeros(0, dtype=oracle.PRED_DTYPE), rate=e["rate"], seed=e["seed"])
        assert n == e["n"]


def _hll_c(oracle, fn, x):
    i, r = ctypes.c_uint32(), ctypes.c_uint32()
    fn(x, 12, ctypes.byref(i), ctypes.byref(r))
    return i.value, r.value


def test_hll_index_rank_worked_values(oracle):
    L = oracle.lib()
    for x, idx, rank in A["hll_i32"]:
        assert oracle.py_hll_i32(x) == (idx, rank), x
        assert _hll_c(oracle, L.oracle_hll_i32, x) == (idx, rank), x
    for x, idx, rank in A["hll_i64"]:
        assert oracle.py_hll_i64(x) == (idx, rank), x
        assert _hll_c(oracle, L.oracle_hll_i64, x) == (idx, rank), x


def test_hll_i64_zero_from_jdk_kat(oracle):
    """int64 HLL of key 0 from the JDK known answer's bits alone (no oracle hash call)."""
    kat = _gold("hash_kats.json")["splitmix64"]["first_nextLong_signed"] & ((1 << 64) - 1)
    idx = kat >> 52
    w = (kat << 12) & ((1 << 64) - 1)
    rank = 64 - w.bit_length() + 1
    assert (idx, rank) == (3618, 5)
    assert oracle.py_hll_i64(0) == (idx, rank)
    assert _hll_c(oracle, oracle.lib().oracle_hll_i64, 0) == (idx, rank)
    # and through a whole probe's registers: one int64 key 0 -> only register 3618 = 5
    _, _, _, regs = oracle.probe([np.zeros(5, dtype=np.int64)], np.zeros(0, dtype=oracle.PRED_DTYPE), hll_cols=[0])
    assert int(regs[0][3618]) == 5 and int(regs[0].sum()) == 5


def test_hll_i32_kat_derived(oracle):
    """int32 (index, rank) of keys 1 and -1 from the MurmurHash3 empty-key vectors' bits."""
    vec = {v["seed"]: v["hash"] for v in _gold("hash_kats.json")["murmur3_x86_32_empty_key"]["vectors"]}
    for x, seed in ((1, 1), (-1, 0xFFFFFFFF)):
        h = vec[seed]
        w = (h << 12) & 0xFFFFFFFF
        assert oracle.py_hll_i32(x) == (h >> 20, 32 - w.bit_length() + 1)


def test_ndv_worked_values(oracle):
    assert abs(oracle.hll_alpha(4096) - A["alpha_4096"]) < 1e-10
    P = np.zeros(0, dtype=oracle.PRED_DTYPE)
    for e in A["ndv_est"]:
        lo, hi = (int(x) for x in e["values"].split(".."))
        col = np.arange(lo, hi + 1, dtype=np.int32)
        _, _, _, regs = oracle.probe([col], P, hll_cols=[0])
        est = oracle.ndv_est(regs[0])
        assert abs(est - e["est"]) <= e["tol"], (e, est)
        if "V" in e:
            assert int((regs[0] == 0).sum()) == e["V"]
            assert est == 4096 * math.log(4096 / e["V"])
