"""Pins for the fp64 oracle (CPU only).

Each test ties an oracle function to something other than itself: a value the
paper prints or that follows from its shapes (tests/golden/, cited), a closed form,
an invariant, a special case that reduces to a textbook/library routine, or brute
force on tiny inputs.  Chosen so that a dropped term, a wrong sign/index or a
transposed operand in the oracle fails at least one of them.
"""
import itertools
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_pairs(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


def _perm(oracle, lat, cfgs, Hh=1):
    """perm[h, p] = token index held at tiled position p (-1 for padded slots)."""
    N = lat[0] * lat[1] * lat[2]
    n = np.arange(N, dtype=np.int64)
    x = np.zeros((Hh, N, 2), dtype=np.uint16)
    x[:, :, 0] = (n & 0xFFFF).astype(np.uint16)
    x[:, :, 1] = (n >> 16).astype(np.uint16)
    xt, cnt, mask = oracle.tile_permute(x, lat, cfgs)
    Hh_, NT, B, _ = xt.shape
    tok = xt[..., 0].astype(np.int64) | (xt[..., 1].astype(np.int64) << 16)
    bits = ((mask[..., :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(Hh_, NT, -1)[..., :B]
    tok = np.where(bits.astype(bool), tok, -1)
    return tok.reshape(Hh_, NT * B), cnt, mask, (NT, B)


def _rand_bf16(rng, shape, scale=1.0):
    from oracle import f64_to_bf16_bits

    return f64_to_bf16_bits(rng.standard_normal(shape) * scale)


# --------------------------------------------------------------------------- grid / tiling


def test_grid_waver_matches_paper_token_count(oracle):
    """245,760 tokens for Waver 720P/241f = padded 61x45x80."""
    g = {r[0]: r[1:] for r in _read_pairs("waver_grid.txt") if r[0] != "hist"}
    for cfg in [(4, 4, 8), (8, 8, 2), (4, 8, 4)]:
        Tp, Hp, Wp, B, NT = oracle.grid((61, 45, 80), [cfg], 1)
        assert (Tp, Hp, Wp) == tuple(int(v) for v in g["padded"])
        assert Tp * Hp * Wp == int(g["tokens"][0]) == 245760
        assert B == 128 and NT == int(g["n_tiles"][0])


def test_waver_tile_count_histogram(oracle):
    rows = _read_pairs("waver_grid.txt")
    hist = {int(r[1]): int(r[2]) for r in rows if r[0] == "hist"}
    real = int([r for r in rows if r[0] == "real_tokens"][0][1])
    lat = (61, 45, 80)
    x = np.zeros((1, 61 * 45 * 80, 1), dtype=np.uint16)
    _, cnt, _ = oracle.tile_permute(x, lat, [(4, 4, 8)])
    vals, counts = np.unique(cnt, return_counts=True)
    assert dict(zip(vals.tolist(), counts.tolist())) == hist
    assert int(cnt.sum()) == real == 219600


def test_tiny_worked_example_golden(oracle):
    perm, cnt, _, (NT, B) = _perm(oracle, (4, 8, 8), [(4, 4, 4)])
    assert (NT, B) == (4, 64)
    for p, n in _read_pairs("tiny_perm.txt"):
        assert perm[0, int(p)] == int(n), p
    assert (cnt == 64).all()


def test_non_divisible_toy_golden(oracle):
    rows = {r[0]: r[1:] for r in _read_pairs("toy_counts.txt")}
    perm, cnt, mask, (NT, B) = _perm(oracle, (3, 5, 6), [(2, 2, 4)])
    assert (NT, B) == (12, 16)
    assert cnt[0].tolist() == [int(v) for v in rows["counts"]]
    last = perm[0, 11 * B:12 * B]
    assert last[0] == int(rows["last_tile_slot0"][0]) and last[1] == int(rows["last_tile_slot1"][0])
    assert (last[2:] == -1).all()


def test_spec_identity_and_box_examples(oracle):
    # SPEC.md:51 shape (1,1,n), cfg (1,1,b) -> identity permutation
    perm, _, _, _ = _perm(oracle, (1, 1, 64), [(1, 1, 16)])
    assert (perm[0] == np.arange(64)).all()
    # SPEC.md:52,62 shape (2,2,2), cfg (2,1,1): tile 0 = {(0,0,0),(1,0,0)} -> tokens 0, 4
    perm, _, _, (NT, B) = _perm(oracle, (2, 2, 2), [(2, 1, 1)])
    assert B == 2 and NT == 4
    assert perm[0, 0] == 0 and perm[0, 1] == 4


@pytest.mark.parametrize("lat,cfgs", [
    ((3, 5, 6), [(2, 2, 4)]),
    ((5, 7, 9), [(2, 4, 2), (4, 2, 2), (1, 4, 4)]),
    ((4, 8, 8), [(4, 4, 4)]),
    ((6, 6, 10), [(4, 4, 8), (8, 4, 4), (4, 8, 4), (8, 8, 2)]),
])
def test_tiling_invariants(oracle, lat, cfgs):
    """Bijection on real slots; every tile an axis-aligned p_t x p_h x p_w box in raster
    box order; slot order raster with t slowest (temporal neighbours are
    p_h*p_w apart); N_T identical across heads (R5)."""
    T, H, W = lat
    Hh = len(cfgs)
    perm, cnt, mask, (NT, B) = _perm(oracle, lat, cfgs, Hh)
    Tp, Hp, Wp, B2, NT2 = oracle.grid(lat, cfgs, Hh)
    assert (B2, NT2) == (B, NT) and Tp * Hp * Wp == NT * B
    for h, (pt, ph, pw) in enumerate(cfgs):
        p = perm[h]
        real = p[p >= 0]
        assert np.array_equal(np.sort(real), np.arange(T * H * W))
        assert int(cnt[h].sum()) == T * H * W
        nbh, nbw = Hp // ph, Wp // pw
        for i in range(NT):
            it, ih, iw = i // (nbh * nbw), (i // nbw) % nbh, i % nbw
            for j in range(B):
                n = p[i * B + j]
                dt, dh, dw = j // (ph * pw), (j // pw) % ph, j % pw
                t, hh, w = it * pt + dt, ih * ph + dh, iw * pw + dw
                if n < 0:
                    assert not (t < T and hh < H and w < W)
                    continue
                assert n == (t * H + hh) * W + w
        # temporal neighbour inside a tile is exactly p_h*p_w slots later
        for i in range(NT):
            for j in range(B - ph * pw):
                a, b = p[i * B + j], p[i * B + j + ph * pw]
                if a >= 0 and b >= 0:
                    assert b - a == H * W


def test_roundtrip_bit_exact(oracle):
    rng = np.random.default_rng(1)
    for lat, cfgs in [((3, 5, 6), [(2, 2, 4)]), ((5, 7, 9), [(2, 4, 2), (4, 2, 2)])]:
        Hh = len(cfgs)
        x = rng.integers(0, 65535, size=(Hh, lat[0] * lat[1] * lat[2], 8), dtype=np.uint16)
        xt, _, _ = oracle.tile_permute(x, lat, cfgs)
        y = oracle.tile_unpermute(xt, lat, cfgs)
        assert np.array_equal(x, y)
        # padded slots are +0
        perm, _, _, _ = _perm(oracle, lat, cfgs, Hh)
        pad = (perm < 0).reshape(xt.shape[:3])
        assert (xt[pad] == 0).all()


def test_k_for_sparsity(oracle):
    # R12 examples: Waver 95% -> 96 of 1920; Wan-1.3B 90% -> 34 of 336; tiny 50% -> 2 of 4
    assert oracle.k_for_sparsity(1920, 0.95) == 96
    assert oracle.k_for_sparsity(336, 0.90) == 34
    assert oracle.k_for_sparsity(4, 0.50) == 2
    assert oracle.k_for_sparsity(1920, 0.0) == 1920
    assert oracle.k_for_sparsity(10, 0.999) == 1


# --------------------------------------------------------------------------- TripPool


def test_trippool_definition_and_special_cases(oracle):
    rng = np.random.default_rng(2)
    lat, cfgs = (3, 5, 6), [(2, 2, 4)]
    x = _rand_bf16(rng, (1, 90, 16), 3.0) | np.uint16(0x8000)  # all values <= 0
    xt, cnt, mask = oracle.tile_permute(x, lat, cfgs)
    z = oracle.trippool(xt, mask)
    xv = oracle.bf16_bits_to_f64(xt)
    perm, _, _, (NT, B) = _perm(oracle, lat, cfgs)
    d = 16
    for i in range(NT):
        valid = perm[0, i * B:(i + 1) * B] >= 0
        rows = xv[0, i][valid]
        assert np.allclose(z[0, i, :d], rows.mean(axis=0), rtol=0, atol=1e-15)
        assert np.array_equal(z[0, i, d:2 * d], rows.max(axis=0))   # Max excludes padded zeros
        assert np.array_equal(z[0, i, 2 * d:], rows.min(axis=0))
    assert (z[..., 2 * d:] <= z[..., :d] + 1e-15).all() and (z[..., :d] <= z[..., d:2 * d] + 1e-15).all()
    # constant tile -> avg = max = min
    xc = np.full((1, 64, 4), 0x4040, dtype=np.uint16)  # 3.0
    xt, _, mk = oracle.tile_permute(xc, (4, 4, 4), [(4, 4, 4)])
    z = oracle.trippool(xt, mk)
    assert (z == 3.0).all()
    # B = 1 -> the token three times
    x1 = _rand_bf16(rng, (1, 8, 4))
    xt, _, mk = oracle.tile_permute(x1, (2, 2, 2), [(1, 1, 1)])
    z = oracle.trippool(xt, mk)
    v = oracle.bf16_bits_to_f64(x1[0])
    assert np.array_equal(z[0], np.concatenate([v, v, v], axis=1))


def test_trippool_empty_tile_is_zero(oracle):
    # mixed configs on a 1x1x4 latent: head 1 (4,1,1) pads T to 4 -> tiles 1.. empty for head 0
    lat, cfgs = (1, 1, 4), [(1, 1, 4), (4, 1, 1)]
    x = np.full((2, 4, 2), 0x3F80, dtype=np.uint16)
    xt, cnt, mask = oracle.tile_permute(x, lat, cfgs)
    z = oracle.trippool(xt, mask)
    assert cnt[0].tolist() == [4, 0, 0, 0] and cnt[1].tolist() == [1, 1, 1, 1]
    assert (z[0, 1:] == 0).all() and (z[0, 0] == 1.0).all()


# --------------------------------------------------------------------------- projection phi


PHI = {1.0: 0.8413447460685429, 2.0: 0.9772498680518208, -1.0: 0.15865525393145707,
       0.5: 0.6914624612740131}  # standard normal CDF (table values)


def test_mlp_gelu_closed_form(oracle):
    """W1 = W2 = I, zero bias -> e = GELU(z) = z * Phi(z) (reading R8)."""
    zs = np.array(list(PHI.keys()) + [0.0])
    din = len(zs)
    z = zs.reshape(1, 1, din)
    eye = np.eye(din, dtype=np.float32)[None]
    e = oracle.mlp(z, eye, np.zeros((1, din), np.float32), eye, np.zeros((1, din), np.float32))
    want = [x * PHI[x] for x in PHI] + [0.0]
    assert np.allclose(e[0, 0], want, rtol=0, atol=1e-15)


def test_mlp_bias_placement_and_zero_weights(oracle):
    din, dh, dl = 6, 5, 4
    z = np.random.default_rng(3).standard_normal((1, 3, din))
    W1 = np.zeros((1, din, dh), np.float32)
    W2 = np.full((1, dh, dl), 0.5, np.float32)
    b1 = np.ones((1, dh), np.float32)          # inside GELU
    b2 = np.arange(dl, dtype=np.float32)[None]  # after the second layer
    e = oracle.mlp(z, W1, b1, W2, b2)
    assert np.allclose(e[0], (dh * 0.5 * 1.0 * PHI[1.0]) + np.arange(dl), rtol=0, atol=1e-14)
    e0 = oracle.mlp(z, W1, np.zeros_like(b1), np.zeros_like(W2), b2)
    assert np.array_equal(e0[0], np.broadcast_to(np.arange(dl, dtype=np.float64), (3, dl)))


def test_mlp_linear_regime_matches_matmul(oracle):
    """Pre-activations > 40 make erf == 1 in fp64, so GELU is the identity and
    e = (z W1 + b1) W2 + b2 exactly as a library matmul computes it (catches a
    transposed W1/W2 or a wrong head offset)."""
    rng = np.random.default_rng(4)
    Hh, NT, din, dh, dl = 2, 5, 6, 7, 3
    z = rng.uniform(1, 2, (Hh, NT, din))
    W1 = rng.uniform(0.5, 1.0, (Hh, din, dh)).astype(np.float32)
    b1 = np.full((Hh, dh), 40.0, np.float32)
    W2 = rng.standard_normal((Hh, dh, dl)).astype(np.float32)
    b2 = rng.standard_normal((Hh, dl)).astype(np.float32)
    e = oracle.mlp(z, W1, b1, W2, b2)
    for h in range(Hh):
        want = (z[h] @ W1[h].astype(np.float64) + b1[h]) @ W2[h].astype(np.float64) + b2[h]
        assert np.allclose(e[h], want, rtol=1e-13, atol=1e-12)


# --------------------------------------------------------------------------- scores


def test_scores_closed_form_and_scale(oracle):
    """W = 0, b2 = c -> S = |c|^2 / sqrt(d') (Eq. 6 scale PAPER.md:268)."""
    for dl in (1, 4, 9):
        c = np.arange(1, dl + 1, dtype=np.float64)
        e = np.broadcast_to(c, (1, 3, dl)).copy()
        s = oracle.scores(e, e, np.ones((1, 3), np.int32))
        assert np.allclose(s, (c @ c) / math.sqrt(dl), rtol=1e-15, atol=0)


def test_scores_matmul_symmetry_rank_and_empty_tiles(oracle):
    rng = np.random.default_rng(5)
    Hh, NT, dl = 2, 12, 3
    eq = rng.standard_normal((Hh, NT, dl))
    ek = rng.standard_normal((Hh, NT, dl))
    cnt = np.full((Hh, NT), 7, np.int32)
    cnt[1, 4] = 0
    s = oracle.scores(eq, ek, cnt)
    for h in range(Hh):
        want = eq[h] @ ek[h].T / math.sqrt(dl)
        ok = cnt[h] > 0
        assert np.allclose(s[h][:, ok], want[:, ok], rtol=1e-14, atol=1e-14)
    assert np.isneginf(s[1, :, 4]).all() and np.isfinite(s[0]).all()
    assert np.linalg.matrix_rank(s[0]) <= dl
    ss = oracle.scores(eq, eq, np.ones((Hh, NT), np.int32))
    assert np.array_equal(ss[0], ss[0].T)


# --------------------------------------------------------------------------- top-k


def test_topk_spec_examples(oracle):
    assert oracle.topk(np.array([[0.1, 0.9, 0.9]]), 1).tolist() == [[1]]
    assert oracle.topk(np.array([[0.3, 0.1, 0.2]]), 3).tolist() == [[0, 1, 2]]
    # all-equal (e.g. zero weights) -> first k indices
    assert oracle.topk(np.zeros((2, 6)), 4).tolist() == [[0, 1, 2, 3]] * 2
    # -inf (empty key tiles) are taken last
    assert oracle.topk(np.array([[-np.inf, 0.0, -np.inf, -5.0]]), 3).tolist() == [[0, 1, 3]]


def test_topk_brute_force_with_ties(oracle):
    rng = np.random.default_rng(6)
    s = rng.integers(-3, 4, size=(40, 17)).astype(np.float64)  # many exact ties
    for k in (1, 5, 16, 17):
        idx = oracle.topk(s, k)
        for r in range(s.shape[0]):
            want = sorted(sorted(range(17), key=lambda j: (-s[r, j], j))[:k])
            assert idx[r].tolist() == want


# --------------------------------------------------------------------------- attention


def _dense_attention_np(q, k, v, scale, key_ok=None):
    """Eq. 1 with the additive-mask form of PAPER.md:140 (key_ok False -> -inf)."""
    l = (q @ k.T) * scale
    if key_ok is not None:
        l = np.where(key_ok, l, -np.inf)
    l = l - l.max(axis=1, keepdims=True)
    p = np.exp(l)
    p /= p.sum(axis=1, keepdims=True)
    return p @ v, p


def _toy_case(oracle, lat, cfgs, d, seed, alpha=4.0):
    rng = np.random.default_rng(seed)
    Hh = len(cfgs)
    N = lat[0] * lat[1] * lat[2]
    u = rng.standard_normal(d)
    u /= np.linalg.norm(u)
    q = _rand_bf16(rng, (Hh, N, d)) if alpha == 0 else oracle.f64_to_bf16_bits(
        alpha * u + rng.standard_normal((Hh, N, d)))
    k = oracle.f64_to_bf16_bits(alpha * u + rng.standard_normal((Hh, N, d)))
    v = _rand_bf16(rng, (Hh, N, d))
    qt, cnt, mask = oracle.tile_permute(q, lat, cfgs)
    kt, _, _ = oracle.tile_permute(k, lat, cfgs)
    vt, _, _ = oracle.tile_permute(v, lat, cfgs)
    return q, k, v, qt, kt, vt, cnt, mask


@pytest.mark.parametrize("lat,cfgs,d", [
    ((4, 8, 8), [(4, 4, 4)], 16),
    ((3, 5, 6), [(2, 2, 4)], 8),
    ((5, 7, 9), [(2, 4, 2), (4, 2, 2), (1, 4, 4)], 8),
])
def test_attention_dense_equals_eq1(oracle, lat, cfgs, d):
    """0% sparsity (k = N_T) equals dense Eq. 1 on the real tokens (north star pin),
    which also fixes padding invariance: padded keys never contribute."""
    q, k, v, qt, kt, vt, cnt, mask = _toy_case(oracle, lat, cfgs, d, 7)
    Hh, NT, B, _ = qt.shape
    idx = np.broadcast_to(np.arange(NT, dtype=np.int32), (Hh, NT, NT)).copy()
    o, lse = oracle.sparse_attn(qt, kt, vt, idx, mask, want_lse=True)
    perm, _, _, _ = _perm(oracle, lat, cfgs, Hh)
    scale = 1 / math.sqrt(d)
    for h in range(Hh):
        qd, kd, vd = (oracle.bf16_bits_to_f64(a[h]) for a in (q, k, v))
        want, _ = _dense_attention_np(qd, kd, vd, scale)
        ll = (qd @ kd.T) * scale
        want_lse = ll.max(1) + np.log(np.exp(ll - ll.max(1, keepdims=True)).sum(1))
        of = o[h].reshape(NT * B, d)
        lf = lse[h].reshape(NT * B)
        real = perm[h] >= 0
        assert np.allclose(of[real], want[perm[h][real]], rtol=0, atol=1e-12)
        assert np.allclose(lf[real], want_lse[perm[h][real]], rtol=0, atol=1e-12)
        assert (of[~real] == 0).all()  # padded query slots -> 0


def test_attention_renormalisation_identity_and_mask_form(oracle):
    """Appendix A.1: sparse probabilities are the dense ones
    renormalised over the kept keys, P~_j = (Z / Z^) P_j; equivalently the additive
    -inf mask form of PAPER.md:140,145."""
    lat, cfgs, d = (3, 5, 6), [(2, 2, 4)], 8
    q, k, v, qt, kt, vt, cnt, mask = _toy_case(oracle, lat, cfgs, d, 8)
    Hh, NT, B, _ = qt.shape
    rng = np.random.default_rng(9)
    kk = 5
    idx = np.stack([np.sort(rng.choice(NT, kk, replace=False)) for _ in range(NT)])[None].astype(np.int32)
    o = oracle.sparse_attn(qt, kt, vt, idx, mask)
    perm, _, _, _ = _perm(oracle, lat, cfgs)
    qd, kd, vd = (oracle.bf16_bits_to_f64(a[0]) for a in (q, k, v))
    N = qd.shape[0]
    tile_of = np.empty(N, dtype=np.int64)
    for p_, n in enumerate(perm[0]):
        if n >= 0:
            tile_of[n] = p_ // B
    _, P = _dense_attention_np(qd, kd, vd, 1 / math.sqrt(d))
    keep = np.zeros((N, N), dtype=bool)
    for n in range(N):
        keep[n] = np.isin(tile_of, idx[0, tile_of[n]])
    renorm = np.where(keep, P, 0.0)
    renorm /= renorm.sum(axis=1, keepdims=True)
    want_a1 = renorm @ vd
    want_mask, _ = _dense_attention_np(qd, kd, vd, 1 / math.sqrt(d), key_ok=keep)
    of = o[0].reshape(NT * B, d)
    real = perm[0] >= 0
    assert np.allclose(of[real], want_a1[perm[0][real]], rtol=0, atol=1e-12)
    assert np.allclose(of[real], want_mask[perm[0][real]], rtol=0, atol=1e-12)


def test_attention_special_cases(oracle):
    rng = np.random.default_rng(10)
    # n = 1 -> output = v
    q = _rand_bf16(rng, (1, 1, 4)); k = _rand_bf16(rng, (1, 1, 4)); v = _rand_bf16(rng, (1, 1, 4))
    args = [oracle.tile_permute(a, (1, 1, 1), [(1, 1, 1)]) for a in (q, k, v)]
    o = oracle.sparse_attn(args[0][0], args[1][0], args[2][0], np.zeros((1, 1, 1), np.int32), args[0][2])
    assert np.array_equal(o[0, 0, 0], oracle.bf16_bits_to_f64(v[0, 0]))
    # V = 1 -> every real output row is 1 (softmax rows sum to 1)
    lat, cfgs, d = (3, 5, 6), [(2, 2, 4)], 8
    _, _, _, qt, kt, _, cnt, mask = _toy_case(oracle, lat, cfgs, d, 11)
    ones = np.full(qt.shape, 0x3F80, dtype=np.uint16)
    NT = qt.shape[1]
    idx = np.stack([np.sort(rng.choice(NT, 4, replace=False)) for _ in range(NT)])[None].astype(np.int32)
    o = oracle.sparse_attn(qt, kt, ones, idx, mask)
    perm, _, _, _ = _perm(oracle, lat, cfgs)
    real = (perm[0] >= 0).reshape(NT, -1)
    assert np.allclose(o[0][real], 1.0, rtol=0, atol=1e-14)
    # identical keys -> uniform weights -> mean of the kept real V rows
    kt_same = np.broadcast_to(kt[:, :1, :1], kt.shape).copy()
    vt = _rand_bf16(rng, qt.shape)
    o = oracle.sparse_attn(qt, kt_same, vt, idx, mask)
    vf = oracle.bf16_bits_to_f64(vt[0])
    for i in range(NT):
        rows = np.concatenate([vf[j][perm[0].reshape(NT, -1)[j] >= 0] for j in idx[0, i]])
        for a in np.nonzero(real[i])[0]:
            assert np.allclose(o[0, i, a], rows.mean(axis=0), rtol=0, atol=1e-14)


def test_attention_list_order_invariance_and_units(oracle):
    lat, cfgs, d = (4, 8, 8), [(4, 4, 4)], 16
    _, _, _, qt, kt, vt, cnt, mask = _toy_case(oracle, lat, cfgs, d, 12)
    idx = np.array([[[0, 2], [1, 3], [0, 3], [2, 3]]], np.int32)
    o = oracle.sparse_attn(qt, kt, vt, idx, mask)
    o2 = oracle.sparse_attn(qt, kt, vt, idx[..., ::-1].copy(), mask)
    assert np.allclose(o, o2, rtol=0, atol=1e-14)
    o3 = oracle.sparse_attn(qt, kt, vt, idx, mask, units=[2])
    assert np.array_equal(o3[0, 2], o[0, 2]) and np.isnan(o3[0, 0]).all()
