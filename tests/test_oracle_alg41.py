"""Pins of the oracle's Algorithm 4.1 (Theorem 4.1).

Hand traces (worked out on paper, recorded in tests/golden/alg41_traces.txt)
and the algorithm's certificate ||A - A~||_F <= eps_g (1 + e_r).
"""
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "alg41_traces.txt")


def _load_traces():
    cases = []
    cur = None
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split("=", 1)
        k = k.strip()
        v = v.strip()
        if k == "case":
            cur = {"name": v}
            cases.append(cur)
        else:
            cur[k] = v
    return cases


def _values(spec: str) -> np.ndarray:
    out = []
    for part in spec.split(","):
        cnt, val = part.split("x")
        out += [float(val)] * int(cnt)
    return np.array(out)


@pytest.mark.parametrize("case", _load_traces(), ids=lambda c: c["name"])
def test_hand_traces(case):
    x = _values(case["values"])
    keep, tau, passes, dropped, hist = O.alg41(x, float(case["eps_g"]), float(case["e_r"]))
    assert passes == int(case["passes"])
    exp_hist = [float(t) for t in case["thresholds"].split(",")] if case["thresholds"] != "-" else []
    assert np.allclose(hist, exp_hist, rtol=1e-15, atol=0)
    assert int(keep.sum()) == int(case["kept"])
    assert dropped == pytest.approx(float(case["dropped"]), rel=1e-14, abs=1e-300)


def test_certificate_and_threshold_property():
    rng = np.random.default_rng(7)
    for _ in range(3000):
        n = int(rng.integers(0, 300))
        mags = 10.0 ** rng.uniform(-22, 0, n)
        x = mags * rng.choice([-1.0, 1.0], n)
        eps_g = 10.0 ** rng.uniform(-20, -2)
        e_r = float(rng.choice([0.01, 0.1, 0.5]))
        keep, tau, passes, dropped, hist = O.alg41(x, eps_g, e_r)
        assert passes < 64  # Theorem 4.1: finite; guard never fires
        assert dropped <= eps_g * (1 + e_r) * (1 + 1e-12)
        # kept set is exactly {|x| > tau} (strict), values untouched
        assert np.array_equal(keep, np.abs(x) > tau)
        # thresholds strictly decrease (Theorem 4.1 proof)
        assert np.all(np.diff(hist) < 0)
        # every threshold is >= eps_g / sqrt(K) (floor lemma used by the GPU path)
        if passes:
            assert hist.min() >= eps_g / np.sqrt(max(n, 1)) * (1 - 1e-12)


def test_eps_zero_keeps_nonzeros():
    x = np.array([0.0, 1e-300, -3.0, 0.0])
    keep, tau, passes, dropped, _ = O.alg41(x, 0.0)
    assert keep.tolist() == [False, True, True, False] and passes == 0 and tau == 0.0


def test_first_pass_unconditional_large_eps():
    # reading R1: the first pass always runs (Theorem 4.1's proof starts from eps_f^(1) = eps_g,
    # P:384), so the certificate ||A - A~||_F <= eps_g (1 + e_r) holds even when
    # eps_g (1 + e_r) >= 1 (the printed scalar b_0 = 1 would drop all of A here: ||A - 0|| = 5.02)
    x = np.array([5.0, 0.5])
    keep, tau, passes, dropped, _ = O.alg41(x, 1.0, 0.1)
    assert passes == 1 and tau == 1.0 and keep.tolist() == [True, False]
    assert dropped == 0.5 <= 1.1


@pytest.mark.parametrize("eps_g", [1.0, 3.0, 40.0, 1e3])
def test_certificate_holds_for_large_eps(eps_g):
    # ||A||_F >> 1 and eps_g (1 + e_r) >= 1: still ||A - A~||_F <= eps_g (1 + e_r)
    rng = np.random.default_rng(int(eps_g))
    x = rng.standard_normal(5000) * rng.choice([1e-3, 1.0, 30.0], 5000)
    keep, tau, passes, dropped, _ = O.alg41(x, eps_g, 0.1)
    assert passes >= 1
    assert np.sqrt(np.sum(x[~keep] ** 2)) == pytest.approx(dropped, rel=1e-12)
    assert dropped <= eps_g * 1.1 * (1 + 1e-12)
    assert np.array_equal(keep, np.abs(x) > tau)


def test_whole_matrix_below_budget_keeps_entries_above_eps():
    # ||A||_F <= eps_g (1 + e_r): one pass at tau = eps_g keeps exactly |x| > eps_g
    x = np.array([0.8, 0.3, -0.2])
    keep, tau, passes, dropped, _ = O.alg41(x, 0.7, 0.5)
    assert passes == 1 and keep.tolist() == [True, False, False]
