"""Sampling on the device vs numpy's Generator.choice on
the same probabilities and seed (the reference's sample, circuit.py:124-133)."""

import numpy as np
import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu


def ref_sample(amps, shots, seed):
    probs = np.abs(amps) ** 2
    return np.random.default_rng(seed).choice(probs.size, size=shots, p=probs / probs.sum())


def assert_same_draws(amps, draws, shots, seed):
    """Every draw equals numpy's (same uniforms, same 'right' cdf search)
    except where the uniform sits within rounding distance of a cdf boundary:
    numpy's sequential float64 cumsum and the device's blocked prefix round
    differently there (no parallel scan reproduces a sequential one).  For each
    disagreement the uniform must lie within 1e-12 of a boundary between the
    two indices (cdf in extended precision)."""
    ref = ref_sample(amps, shots, seed)
    u = np.random.default_rng(seed).random(shots)
    probs = (np.abs(amps) ** 2).astype(np.longdouble)
    cdf = np.cumsum(probs) / probs.sum()
    bad = np.nonzero(draws != ref)[0]
    for k in bad:
        lo, hi = sorted((int(draws[k]), int(ref[k])))
        assert np.min(np.abs(cdf[lo:hi] - u[k])) <= 1e-12, (k, lo, hi, u[k])
    assert bad.size <= max(2, shots // 1000)


@pytest.mark.parametrize("n,p", [(3, 1), (10, 2), (16, 3), (20, 2)])
def test_sample_matches_numpy(n, p):
    g = Q.random_regular_graph(n, 3, seed=n) if n > 3 else Q.complete_graph(3)
    s = Q.simulate(g, Q.params_from_seed(p, n), "bitwise", exact=True)
    draws = Q.sample(s, 20000, seed=7)
    assert_same_draws(s.amps, draws, 20000, 7)
    assert draws.min() >= 0 and draws.max() < (1 << n)


def test_sample_complemented_state():
    # beta near pi: the fast schedule stores the state index-complemented
    g = Q.random_regular_graph(14, 3, seed=1)
    s = Q.simulate(g, Q.QaoaParams((0.4,), (3.0,)), "bitwise")
    draws = Q.sample(s, 5000, seed=3)
    assert_same_draws(s.amps, draws, 5000, 3)


def test_sample_kats():
    amps = np.zeros(4, dtype=np.complex128)
    amps[0b10] = 1.0
    assert set(Q.sample(Q.StateVector(2, amps), shots=50, seed=1).tolist()) == {0b10}
    draws = Q.sample(Q.init_uniform(1), shots=10000, seed=3)
    assert 0.47 <= np.mean(draws == 0) <= 0.53
    with pytest.raises(ValueError):
        Q.sample(Q.init_uniform(2), shots=0)
    with pytest.raises(ValueError, match="normalized"):
        Q.sample(Q.StateVector(2, np.full(4, 0.6, dtype=np.complex128)), shots=10)
    s = Q.init_uniform(4)
    np.testing.assert_array_equal(Q.sample(s, 100, seed=9), Q.sample(s, 100, seed=9))
