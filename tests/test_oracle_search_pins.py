"""Pins for the oracle's head-aware tiling search (Alg. 1, Eq. 8-9) -- CPU only.

* Omega (Eq. 8) against the closed-form count of ordered factorisations.
* The error cube E against an independent numpy re-derivation that never calls the
  oracle's tiling: tile ids from the box formula, dense softmax, block max, Top-k by
  lexsort, masked softmax, squared Frobenius error.
* k_top >= N_T for every candidate -> sparse == dense -> E = 0.
* A constructed "line-local" head whose attention stays inside each (t, h) row: the
  tiling whose boxes are exactly those rows reproduces full attention with k_top = 1, so it
  is the unique argmin with E ~ 0 while every other candidate has a large error.
"""
import math

import numpy as np
import pytest

from test_oracle_pins import _rand_bf16


def test_omega_counts_and_members(oracle):
    for B, want in ((128, 36), (64, 28), (8, 10), (12, 18), (1, 1)):
        om = oracle.omega(B)
        assert len(om) == want and len(set(om)) == want  # prod over primes C(a+2, 2)
        assert all(a * b * c == B for a, b, c in om)


def _numpy_errors(q, k, v, lat, cands, k_top):
    """Alg. 1 re-derived with numpy only (no oracle tiling or attention routine)."""
    T, H, W = lat
    Hh, N, d = q.shape
    t, h, w = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    t, h, w = t.ravel(), h.ravel(), w.ravel()  # raster order n = (t*H + h)*W + w
    E = np.zeros((Hh, len(cands)))
    for hh in range(Hh):
        qd, kd, vd = (a[hh] for a in (q, k, v))
        l = (qd @ kd.T) / math.sqrt(d)
        A = np.exp(l - l.max(1, keepdims=True))
        A /= A.sum(1, keepdims=True)
        o_fu = A @ vd
        for c, (pt, ph, pw) in enumerate(cands):
            Hp, Wp = -(-H // ph) * ph, -(-W // pw) * pw
            Tp = -(-T // pt) * pt
            NT = Tp * Hp * Wp // (pt * ph * pw)
            tile = ((t // pt) * (Hp // ph) + h // ph) * (Wp // pw) + w // pw
            S = np.full((NT, NT), -np.inf)
            for i in range(NT):
                ui = tile == i
                for j in range(NT):
                    vj = tile == j
                    if vj.any():
                        S[i, j] = A[np.ix_(ui, vj)].max() if ui.any() else 0.0
            kk = min(k_top, NT)
            keep = np.zeros((NT, NT), bool)
            for i in range(NT):
                order = np.lexsort((np.arange(NT), -S[i]))
                keep[i, order[:kk]] = True
            allowed = keep[tile][:, tile]  # token-level mask
            lm = np.where(allowed, l, -np.inf)
            P = np.exp(lm - lm.max(1, keepdims=True))
            P /= P.sum(1, keepdims=True)
            E[hh, c] = ((o_fu - P @ vd) ** 2).sum()
    return E


@pytest.mark.parametrize("lat,k_top", [((3, 4, 6), 2), ((2, 5, 4), 3)])
def test_search_errors_match_numpy_rederivation(oracle, lat, k_top):
    rng = np.random.default_rng(31)
    Hh, d = 2, 8
    N = lat[0] * lat[1] * lat[2]
    u = rng.standard_normal(d)
    q = oracle.f64_to_bf16_bits(3 * u + rng.standard_normal((Hh, N, d)))
    k = oracle.f64_to_bf16_bits(3 * u + rng.standard_normal((Hh, N, d)))
    v = _rand_bf16(rng, (Hh, N, d))
    cands = oracle.omega(8)
    E = oracle.tiling_search_errors(q, k, v, lat, k_top, cands, nthreads=2)
    want = _numpy_errors(*(oracle.bf16_bits_to_f64(a) for a in (q, k, v)), lat, cands, k_top)
    assert np.allclose(E, want, rtol=1e-9, atol=1e-14)
    assert (E > 0).any()


def test_search_dense_budget_gives_zero_error(oracle):
    rng = np.random.default_rng(32)
    lat, d = (2, 4, 4), 8
    N = 32
    q, k, v = (_rand_bf16(rng, (1, N, d)) for _ in range(3))
    E = oracle.tiling_search_errors(q, k, v, lat, 10 ** 6, oracle.omega(8), nthreads=2)
    assert np.abs(E).max() < 1e-24


def line_local_qkv(oracle, lat, d, Hh=1, seed=33, c=8.0):
    """q = k = c * e_line(t, h): attention stays inside each (t, h) row of the latent."""
    T, H, W = lat
    assert T * H <= d
    rng = np.random.default_rng(seed)
    N = T * H * W
    line = np.repeat(np.arange(T * H), W)
    x = np.zeros((Hh, N, d))
    x[:, np.arange(N), line] = c
    q = oracle.f64_to_bf16_bits(x)
    v = _rand_bf16(rng, (Hh, N, d))
    return q, q.copy(), v


def test_search_line_local_head_picks_row_tiles(oracle):
    lat, d = (2, 4, 8), 16
    q, k, v = line_local_qkv(oracle, lat, d)
    cands = oracle.omega(8)
    E = oracle.tiling_search_errors(q, k, v, lat, 1, cands, nthreads=2)
    best = int(np.argmin(E[0]))
    assert cands[best] == (1, 1, 8)
    assert E[0, best] < 1e-8
    others = np.delete(E[0], best)
    assert others.min() > 1e-2
