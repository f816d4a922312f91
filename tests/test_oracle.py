"""CPU tests: the oracle restatement is pinned against the reference.

* golden vectors produced by the unmodified reference (tests/golden/make_golden.py)
* the reference's own known-answer tests restated (test_grid_fourier.cpp,
  test_regularizer.cpp), applied to the oracle
"""
import numpy as np
import pytest

from oracle_lib import Oracle, make_cfg
from paper_1905_13408_b200 import synth
from golden.make_golden import CONFIGS, random_accumulator, random_volume, sha

G = np.load(__import__("pathlib").Path(__file__).parent / "golden" / "reference_golden.npz")


@pytest.fixture(scope="module")
def O():
    return Oracle()


def test_fft_matches_reference_golden(O):
    x = random_volume(6, 3)
    assert sha(x) == str(G["fft6_x_sha"])
    np.testing.assert_allclose(O.fft3(x), G["fft6"], atol=1e-12)
    # and an independent FFT (numpy pocketfft) agrees with the convention
    np.testing.assert_allclose(G["fft6"], np.fft.fftn(x), atol=1e-12)
    np.testing.assert_allclose(G["fft6c"], np.fft.fftn(synth.halfshift3(x)), atol=1e-12)


@pytest.mark.parametrize("n", [4, 6, 8, 10, 12, 18])
def test_fft_kats(O, n):
    """test_grid_fourier.cpp:29-96: delta -> ones, DC, Plancherel."""
    d = np.zeros((n, n, n))
    d[0, 0, 0] = 1.0
    np.testing.assert_allclose(O.fft3(d), np.ones((n, n, n)), atol=1e-12)
    x = np.random.default_rng(n).standard_normal((n, n, n))
    F = O.fft3(x)
    np.testing.assert_allclose(F, np.fft.fftn(x), atol=1e-10 * np.abs(F).max())
    assert abs((np.abs(F) ** 2).sum() / n**3 - (x * x).sum()) < 1e-10 * (x * x).sum()


@pytest.mark.parametrize("n,seed", [(6, 11), (8, 12)])
def test_random_accumulator_golden(O, n, seed):
    w, y = random_accumulator(n, seed)
    x = random_volume(n, seed + 100)
    assert sha(w, y, x) == str(G[f"racc{n}_sha"])
    rc, sy, sn = O.scale_data(w, y)
    assert rc == 0
    np.testing.assert_allclose([sy, sn], G[f"racc{n}_scales"], rtol=1e-12)
    rc, g = O.data_gradient(w, y, x)
    assert rc == 0
    np.testing.assert_allclose(g, G[f"racc{n}_dgrad"], atol=1e-13)
    assert abs(O.symmetry_residue(w, y) - G[f"racc{n}_resid"][0]) < 1e-15


@pytest.mark.parametrize("n", [16, 32])
def test_m_step_traces_golden(O, n):
    p = synth.synthetic_problem(n)
    k = f"prob{n}"
    assert sha(p.weight, p.numerator, p.x0) == str(G[k + "_sha"])
    rc, sy, sn = O.scale_data(p.weight, p.numerator)
    np.testing.assert_allclose([sy, sn], G[k + "_scales"], rtol=1e-12)
    rc, cfg = O.derive_config(sy, sn, p.eps, p.eps_prime)
    assert rc == 0
    np.testing.assert_allclose([cfg.alpha, cfg.beta, cfg.gamma, cfg.eps, cfg.eps_prime, cfg.mu],
                               G[k + "_cfg"], rtol=1e-13)
    rc, g = O.data_gradient(p.weight, p.numerator, p.x0)
    np.testing.assert_allclose(g, G[k + "_dgrad"], atol=1e-12)
    xp = p.x0 + 0.05 * random_volume(n, 7)
    rc, obj = O.penalized_objective(p.weight, p.numerator, xp, cfg, p.x0, p.x0)
    np.testing.assert_allclose(obj, G[k + "_obj"], rtol=1e-11)
    for name, extra in CONFIGS.items():
        tr_ref = G[f"{k}_{name}_trace"]
        c = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                     eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=len(tr_ref),
                     fixed_step=float(G[f"{k}_{name}_fixed_step"][0]))
        for kk, vv in extra.items():
            setattr(c, kk, vv)
        rc, x, tr = O.m_step(p.weight, p.numerator, p.x0, p.x0, c)
        assert rc == 0
        np.testing.assert_allclose(tr, tr_ref, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(x, G[f"{k}_{name}_x"], atol=1e-12)


def test_prox_kat(O):
    """test_regularizer.cpp:244-256 values, |x| == t lands at zero."""
    v = np.array([0.5, -2.0, 0.0, 3.25, -0.75, 1.0, -1.0, 0.2]).reshape(2, 2, 2)
    t = np.array([1.0, 0.5, 0.7, 0.25, 0.75, 1.0, 0.5, 0.0]).reshape(2, 2, 2)
    got = O.prox_l1(v, t).reshape(-1)
    np.testing.assert_array_equal(got, [0.0, -1.5, 0.0, 3.0, 0.0, 0.0, -0.5, 0.2])


def test_gradient_adjointness(O):
    """test_grid_fourier.cpp:199-217 (replicate)."""
    rng = np.random.default_rng(31)
    x = rng.standard_normal((6, 6, 6))
    g = [rng.standard_normal((6, 6, 6)) for _ in range(3)]
    d = O.discrete_gradient(x)
    lhs = sum((a * b).sum() for a, b in zip(d, g))
    rhs = (x * O.gradient_adjoint(*g)).sum()
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)


def test_unregularized_converges_to_target(O):
    """test_regularizer.cpp:331-345 restated on the oracle."""
    n = 6
    w = synth.symmetric_weight(n, 21)
    target = random_volume(n, 22)
    y = w * synth.fft3_centered(target)
    cfg = make_cfg(inner_iters=50)
    z = np.zeros((n, n, n))
    rc, x, _ = O.m_step(w, y, z, z, cfg, trace=False)
    assert rc == 0 and np.abs(x - target).max() < 1e-6


def test_error_codes(O):
    n = 6
    w = synth.symmetric_weight(n, 1)
    y = w * synth.fft3_centered(random_volume(n, 2))
    x = random_volume(n, 3)
    assert O.data_gradient(w, y, x, finalized=False)[0] == 3
    yb = y.copy()
    yb[0, 0, 1] += 1.0  # break Friedel symmetry
    assert O.data_gradient(w, yb, x)[0] == 3
    assert O.m_step(w, y, x, x, make_cfg(alpha=-1.0))[0] == 1
    assert O.m_step(w, y, x, x, make_cfg(inner_iters=0))[0] == 1
    assert O.m_step(w, y, x, x, make_cfg(step_rule=1, fixed_step=0.0))[0] == 1
    assert O.derive_config(0.0, 5.0, 0.1, 0.05)[0] == 7
