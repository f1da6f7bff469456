"""Pins for the oracle's target tile scores (Eq. 4) and tile recall (Eq. 3) -- CPU only.

S_tgt is pinned to a brute-force numpy construction that does NOT go through tiling:
the dense softmax A* over the untiled tokens (textbook Eq. 1), max-pooled over the
token sets that tests/golden/tiny_perm.txt-style permutations assign to each tile,
plus closed forms (uniform attention -> 1/N, a single tile -> max_uv A*, rows of a
one-hot attention), and invariants.  Recall is pinned by hand-counted examples.
"""
import math

import numpy as np
import pytest

from test_oracle_pins import _dense_attention_np, _perm, _rand_bf16, _toy_case


def _brute_target(oracle, q, k, lat, cfgs, d):
    """max over (u in tile i, v in tile j) of the dense softmax, from untiled tokens."""
    Hh = q.shape[0]
    perm, cnt, mask, (NT, B) = _perm(oracle, lat, cfgs, Hh)
    out = np.zeros((Hh, NT, NT))
    for h in range(Hh):
        qd, kd = oracle.bf16_bits_to_f64(q[h]), oracle.bf16_bits_to_f64(k[h])
        _, P = _dense_attention_np(qd, kd, kd, 1 / math.sqrt(d))
        tiles = perm[h].reshape(NT, B)
        for i in range(NT):
            qi = tiles[i][tiles[i] >= 0]
            for j in range(NT):
                kj = tiles[j][tiles[j] >= 0]
                if len(kj) == 0:
                    out[h, i, j] = -np.inf
                elif len(qi) == 0:
                    out[h, i, j] = 0.0
                else:
                    out[h, i, j] = P[np.ix_(qi, kj)].max()
    return out


@pytest.mark.parametrize("lat,cfgs,d", [
    ((4, 8, 8), [(4, 4, 4)], 16),
    ((3, 5, 6), [(2, 2, 4)], 8),
    ((5, 7, 9), [(2, 4, 2), (4, 2, 2), (1, 4, 4)], 8),
])
def test_target_equals_maxpooled_dense_softmax(oracle, lat, cfgs, d):
    """Eq. 4 against brute force from the untiled dense softmax."""
    q, k, _, qt, kt, _, cnt, mask = _toy_case(oracle, lat, cfgs, d, 21)
    s = oracle.target_scores(qt, kt, mask, nthreads=2)
    want = _brute_target(oracle, q, k, lat, cfgs, d)
    fin = np.isfinite(want)
    assert np.array_equal(fin, np.isfinite(s))
    assert np.allclose(s[fin], want[fin], rtol=1e-12, atol=1e-15)


def test_target_closed_forms(oracle):
    rng = np.random.default_rng(22)
    lat, cfgs, d = (3, 5, 6), [(2, 2, 4)], 8
    N = 90
    # identical keys -> A* uniform = 1/N over real keys, every non-empty block = 1/N
    q = _rand_bf16(rng, (1, N, d))
    k = np.broadcast_to(_rand_bf16(rng, (1, 1, d)), (1, N, d)).copy()
    qt, cnt, mask = oracle.tile_permute(q, lat, cfgs)
    kt, _, _ = oracle.tile_permute(k, lat, cfgs)
    s = oracle.target_scores(qt, kt, mask)
    real_q = cnt[0] > 0
    assert np.allclose(s[0][real_q], 1.0 / N, rtol=1e-13, atol=0)
    # a single tile holding everything -> S_tgt = max_uv A*_uv (a 1x1 matrix)
    lat1, cfg1 = (2, 2, 4), [(2, 2, 4)]
    q, k, _, qt, kt, _, cnt, mask = _toy_case(oracle, lat1, cfg1, d, 23)
    s = oracle.target_scores(qt, kt, mask)
    qd, kd = oracle.bf16_bits_to_f64(q[0]), oracle.bf16_bits_to_f64(k[0])
    _, P = _dense_attention_np(qd, kd, kd, 1 / math.sqrt(d))
    assert s.shape == (1, 1, 1) and abs(s[0, 0, 0] - P.max()) < 1e-15
    # near one-hot attention: q = c * k_n for a large c -> query n's row peaks at key n,
    # so the block holding (n, n) scores ~1 and every other block of that row ~0
    lat, cfgs, d = (2, 4, 4), [(1, 2, 2)], 32
    N = 32
    kf = np.linalg.qr(rng.standard_normal((d, d)))[0][:N]  # orthonormal keys
    k = oracle.f64_to_bf16_bits(kf[None])
    q = oracle.f64_to_bf16_bits(400.0 * kf[None])
    qt, cnt, mask = oracle.tile_permute(q, lat, cfgs)
    kt, _, _ = oracle.tile_permute(k, lat, cfgs)
    s = oracle.target_scores(qt, kt, mask)
    NT = s.shape[1]
    assert np.allclose(np.diag(s[0]), 1.0, atol=1e-6)
    assert (s[0][~np.eye(NT, dtype=bool)] < 1e-6).all()


def test_target_invariants_and_units(oracle):
    lat, cfgs, d = (5, 7, 9), [(2, 4, 2), (4, 2, 2)], 8
    q, k, _, qt, kt, _, cnt, mask = _toy_case(oracle, lat, cfgs, d, 24)
    s = oracle.target_scores(qt, kt, mask)
    Hh, NT, _ = s.shape
    fin = np.isfinite(s)
    # probabilities: in (0, 1] on real query tiles, 0 on empty ones; -inf exactly on
    # empty key tiles; row max >= 1/(#real keys)
    assert np.array_equal(~fin, np.broadcast_to((cnt == 0)[:, None, :], s.shape))
    rq = np.broadcast_to((cnt > 0)[:, :, None], s.shape)
    assert ((s[fin & rq] > 0) & (s[fin & rq] <= 1)).all()
    assert (s[fin & ~rq] == 0).all()
    for h in range(Hh):
        for i in range(NT):
            if cnt[h, i]:
                assert s[h, i][fin[h, i]].max() >= 1.0 / cnt[h].sum() - 1e-15
    # the result is invariant to the order of slots within a tile (max is order-free)
    rng = np.random.default_rng(25)
    B = qt.shape[2]
    sl = rng.permutation(B)
    # permute slots of every tile consistently in q, k and the mask bits
    bits = ((mask[..., :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(Hh, NT, -1)[..., :B]
    bits = bits[..., sl]
    m2 = np.zeros_like(mask)
    for b in range(B):
        m2[..., b // 32] |= (bits[..., b].astype(np.uint32) << np.uint32(b % 32))
    s2 = oracle.target_scores(qt[:, :, sl].copy(), kt[:, :, sl].copy(), m2)
    assert np.array_equal(np.isfinite(s2), fin)
    assert np.allclose(s2[fin], s[fin], rtol=1e-12, atol=0)
    # units subset computes only those rows
    s3 = oracle.target_scores(qt, kt, mask, units=[NT + 1])
    assert np.array_equal(s3[1, 1], s[1, 1]) and np.isnan(s3[0]).all()


def test_recall_hand_counted(oracle):
    """Eq. 3: mean_i |S_sp,i & S_fu,i| / k."""
    sp = np.array([[0, 1, 2], [3, 4, 5], [0, 2, 4], [1, 3, 5]], np.int32)
    fu = np.array([[0, 1, 2], [0, 1, 2], [4, 2, 9], [5, 1, 7]], np.int32)
    # per row: 3/3, 0/3, 2/3, 2/3
    assert abs(oracle.recall(sp, fu) - (1 + 0 + 2 / 3 + 2 / 3) / 4) < 1e-15
    # rows with no real token are excluded (R4)
    cnt = np.array([5, 0, 5, 0], np.int32)
    assert abs(oracle.recall(sp, fu, cnt) - (1 + 2 / 3) / 2) < 1e-15
    # k = N_T -> recall 1 for any lists; identical lists -> 1; disjoint -> 0
    full = np.tile(np.arange(6, dtype=np.int32), (3, 1))
    assert oracle.recall(full, full[:, ::-1].copy()) == 1.0
    assert oracle.recall(sp, sp) == 1.0
    assert oracle.recall(np.array([[0, 1]], np.int32), np.array([[2, 3]], np.int32)) == 0.0


def test_recall_of_target_topk_is_one(oracle):
    """The oracle mask M~* = TopK(S_tgt) recalls itself; S_pred = S_tgt gives recall 1 and
    a random list has the expected recall ~ k / N_T on a large row count."""
    lat, cfgs, d = (4, 8, 8), [(1, 2, 4)], 16
    q, k, _, qt, kt, _, cnt, mask = _toy_case(oracle, lat, cfgs, d, 26)
    s = oracle.target_scores(qt, kt, mask)
    NT = s.shape[1]
    kk = 5
    star = oracle.topk(s, kk)
    assert oracle.recall(star, star, cnt) == 1.0
    rng = np.random.default_rng(27)
    rnd = np.stack([np.sort(rng.choice(NT, kk, replace=False)) for _ in range(4000)]).astype(np.int32)
    ref = np.tile(star[0, 0], (4000, 1))
    assert abs(oracle.recall(rnd, ref) - kk / NT) < 0.02
