"""fp64 CPU oracle for the Veda tile-sparse attention hot path (arXiv 2605.30325).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path in ``paper_2605_30325_b200``
and never imports it; the C source ``veda_oracle.c`` is written from PAPER.md
alone (each routine cites its passage).

Parity pins (tests/test_oracle_pins.py) check every function against values
and properties fixed by the paper and by mathematics.  No function here is
"parity unpinned".

Array conventions (numpy):
  * bf16 tensors are ``np.uint16`` bit patterns;
  * tiled tensors are ``[Hh, N_T, B, d]``; masks ``[Hh, N_T, ceil(B/32)]`` uint32;
  * everything floating is fp64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "veda_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, IEEE semantics, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.vo_grid.argtypes = [i32, i32, i32, P, i32, P]
        lib.vo_tile_permute.argtypes = [P, i64, i64, i32, i32, i32, P, i32, i32, P, P, P]
        lib.vo_tile_unpermute.argtypes = [P, i32, i32, i32, P, i32, i32, P, i64, i64]
        lib.vo_trippool.argtypes = [P, P, i32, i64, i32, i32, P]
        lib.vo_trippool.restype = None
        lib.vo_mlp.argtypes = [P, i32, i64, i32, i32, i32, P, P, P, P, P]
        lib.vo_mlp.restype = None
        lib.vo_scores.argtypes = [P, P, P, i32, i64, i32, P]
        lib.vo_scores.restype = None
        lib.vo_topk.argtypes = [P, i64, i64, i32, P]
        lib.vo_sparse_attn.argtypes = [P, P, P, P, P, i32, i64, i32, i32, i32, dbl, P, i64, P, P, i32]
        lib.vo_target_scores.argtypes = [P, P, P, i32, i64, i32, i32, dbl, P, i64, P, i32]
        lib.vo_target_scores.restype = None
        lib.vo_recall.argtypes = [P, P, P, i64, i32]
        lib.vo_recall.restype = dbl
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _cfg_array(cfgs, Hh):
    c = np.asarray(cfgs, dtype=np.int32).reshape(-1, 3)
    if c.shape[0] == 1 and Hh > 1:
        c = np.repeat(c, Hh, axis=0)
    assert c.shape[0] == Hh
    return np.ascontiguousarray(c)


def grid(lat, cfgs, Hh: int):
    """(T', H', W', B, N_T) of the padded grid.  PAPER.md:143-145, 288-294, 471."""
    c = _cfg_array(cfgs, Hh)
    out = np.zeros(5, dtype=np.int64)
    rc = _load().vo_grid(int(lat[0]), int(lat[1]), int(lat[2]), _p(c), Hh, _p(out))
    if rc:
        raise ValueError(f"invalid latent/config (code {rc})")
    return tuple(int(v) for v in out)


def k_for_sparsity(n_tiles: int, sparsity: float) -> int:
    """Reading R12: k = floor((1-s) N_T + 1/2), clamped to [1, N_T]."""
    import math
    k = math.floor((1.0 - sparsity) * n_tiles + 0.5)
    return max(1, min(n_tiles, k))


def tile_permute(x: np.ndarray, lat, cfgs):
    """x: [Hh, N, d] uint16 -> (xt [Hh,N_T,B,d] uint16, cnt [Hh,N_T] int32, mask)."""
    x = np.ascontiguousarray(x, dtype=np.uint16)
    Hh, N, d = x.shape
    assert N == lat[0] * lat[1] * lat[2]
    c = _cfg_array(cfgs, Hh)
    _, _, _, B, NT = grid(lat, c, Hh)
    xt = np.empty((Hh, NT, B, d), dtype=np.uint16)
    cnt = np.empty((Hh, NT), dtype=np.int32)
    mask = np.empty((Hh, NT, (B + 31) // 32), dtype=np.uint32)
    rc = _load().vo_tile_permute(_p(x), N * d, d, lat[0], lat[1], lat[2], _p(c), Hh, d,
                                 _p(xt), _p(cnt), _p(mask))
    assert rc == 0
    return xt, cnt, mask


def tile_unpermute(xt: np.ndarray, lat, cfgs):
    """xt [Hh,N_T,B,d] uint16 -> x [Hh,N,d] uint16 (padded slots dropped)."""
    xt = np.ascontiguousarray(xt, dtype=np.uint16)
    Hh, NT, B, d = xt.shape
    c = _cfg_array(cfgs, Hh)
    N = lat[0] * lat[1] * lat[2]
    x = np.zeros((Hh, N, d), dtype=np.uint16)
    rc = _load().vo_tile_unpermute(_p(xt), lat[0], lat[1], lat[2], _p(c), Hh, d, _p(x), N * d, d)
    assert rc == 0
    return x


def trippool(xt: np.ndarray, mask: np.ndarray):
    """Eq. 5: z = Avg (+) Max (+) Min over real slots -> [Hh, N_T, 3d] fp64."""
    xt = np.ascontiguousarray(xt, dtype=np.uint16)
    mask = np.ascontiguousarray(mask, dtype=np.uint32)
    Hh, NT, B, d = xt.shape
    z = np.empty((Hh, NT, 3 * d), dtype=np.float64)
    _load().vo_trippool(_p(xt), _p(mask), Hh, NT, B, d, _p(z))
    return z


def mlp(z: np.ndarray, W1, b1, W2, b2):
    """Eq. 6 projection phi: e = GELU(z W1 + b1) W2 + b2 per head -> fp64."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    Hh, NT, din = z.shape
    W1 = np.ascontiguousarray(W1, dtype=np.float32)
    W2 = np.ascontiguousarray(W2, dtype=np.float32)
    b1 = np.ascontiguousarray(b1, dtype=np.float32)
    b2 = np.ascontiguousarray(b2, dtype=np.float32)
    dh, dl = W1.shape[-1], W2.shape[-1]
    assert W1.shape == (Hh, din, dh) and W2.shape == (Hh, dh, dl)
    assert b1.shape == (Hh, dh) and b2.shape == (Hh, dl)
    e = np.empty((Hh, NT, dl), dtype=np.float64)
    _load().vo_mlp(_p(z), Hh, NT, din, dh, dl, _p(W1), _p(b1), _p(W2), _p(b2), _p(e))
    return e


def scores(eq: np.ndarray, ek: np.ndarray, cnt_k: np.ndarray):
    """Eq. 6 scores S_ij = e_q,i . e_k,j / sqrt(d'); -inf for empty key tiles."""
    eq = np.ascontiguousarray(eq, dtype=np.float64)
    ek = np.ascontiguousarray(ek, dtype=np.float64)
    cnt_k = np.ascontiguousarray(cnt_k, dtype=np.int32)
    Hh, NT, dl = eq.shape
    s = np.empty((Hh, NT, NT), dtype=np.float64)
    _load().vo_scores(_p(eq), _p(ek), _p(cnt_k), Hh, NT, dl, _p(s))
    return s


def topk(s: np.ndarray, k: int):
    """Exactly-k per row, ties to the lower index, ascending output -> int32."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    shape = s.shape
    ncols = shape[-1]
    rows = int(np.prod(shape[:-1]))
    idx = np.empty(shape[:-1] + (k,), dtype=np.int32)
    rc = _load().vo_topk(_p(s), rows, ncols, k, _p(idx))
    if rc:
        raise ValueError("k out of range")
    return idx


def sparse_attn(qt, kt, vt, idx, mask, scale: float = 0.0, units=None, nthreads: int | None = None,
                want_lse: bool = False):
    """Eq. 2 over the kept tiles of idx.  Returns o [Hh,N_T,B,d] fp64 (and lse).

    ``units``: optional iterable of unit ids ``h*N_T + i``; only those are computed
    (others are left as NaN so accidental use is visible).
    """
    qt = np.ascontiguousarray(qt, dtype=np.uint16)
    kt = np.ascontiguousarray(kt, dtype=np.uint16)
    vt = np.ascontiguousarray(vt, dtype=np.uint16)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    mask = np.ascontiguousarray(mask, dtype=np.uint32)
    Hh, NT, B, d = qt.shape
    k = idx.shape[-1]
    o = np.full((Hh, NT, B, d), np.nan, dtype=np.float64)
    lse = np.full((Hh, NT, B), np.nan, dtype=np.float64) if want_lse else None
    if units is not None:
        u = np.ascontiguousarray(np.asarray(list(units), dtype=np.int64))
        up, nu = _p(u), len(u)
    else:
        up, nu = None, 0
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    rc = _load().vo_sparse_attn(_p(qt), _p(kt), _p(vt), _p(idx), _p(mask), Hh, NT, B, d, k,
                                float(scale), up, nu, _p(o), _p(lse) if lse is not None else None,
                                int(nthreads))
    if rc:
        raise ValueError("k out of range")
    return (o, lse) if want_lse else o


def target_scores(qt, kt, mask, scale: float = 0.0, units=None, nthreads: int | None = None):
    """Eq. 4: S_tgt_ij = max over the (i, j) tile block of A* = softmax(Q K^T / sqrt(d)).
    Returns [Hh, N_T, N_T] fp64 (rows of units not listed are NaN)."""
    qt = np.ascontiguousarray(qt, dtype=np.uint16)
    kt = np.ascontiguousarray(kt, dtype=np.uint16)
    mask = np.ascontiguousarray(mask, dtype=np.uint32)
    Hh, NT, B, d = qt.shape
    s = np.full((Hh, NT, NT), np.nan, dtype=np.float64)
    if units is not None:
        u = np.ascontiguousarray(np.asarray(list(units), dtype=np.int64))
        up, nu = _p(u), len(u)
    else:
        up, nu = None, 0
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    _load().vo_target_scores(_p(qt), _p(kt), _p(mask), Hh, NT, B, d, float(scale), up, nu, _p(s), int(nthreads))
    return s


def recall(idx_sp, idx_fu, cnt=None) -> float:
    """Eq. 3: mean over (real) query tiles of |S_sp & S_fu| / k."""
    a = np.ascontiguousarray(idx_sp, dtype=np.int32)
    b = np.ascontiguousarray(idx_fu, dtype=np.int32)
    k = a.shape[-1]
    rows = int(np.prod(a.shape[:-1]))
    c = np.ascontiguousarray(cnt, dtype=np.int32) if cnt is not None else None
    return float(_load().vo_recall(_p(a), _p(b), _p(c) if c is not None else None, rows, k))


def omega(B: int):
    """Eq. 8 search space (Alg. 1 l.640): all (p_t, p_h, p_w) in N^3 with
    p_t p_h p_w = B, in lexicographic order."""
    out = []
    for pt in range(1, B + 1):
        if B % pt:
            continue
        for ph in range(1, B // pt + 1):
            if (B // pt) % ph:
                continue
            out.append((pt, ph, B // (pt * ph)))
    return out


def token_index(lat, cfgs, Hh: int):
    """perm [Hh, N_T*B]: token index held by each tiled slot (-1 for padding), obtained by
    tiling a payload of token ids with vo_tile_permute."""
    N = lat[0] * lat[1] * lat[2]
    n = np.arange(N, dtype=np.int64)
    x = np.zeros((Hh, N, 2), dtype=np.uint16)
    x[:, :, 0] = (n & 0xFFFF).astype(np.uint16)
    x[:, :, 1] = (n >> 16).astype(np.uint16)
    xt, cnt, mask = tile_permute(x, lat, cfgs)
    Hh_, NT, B, _ = xt.shape
    tok = xt[..., 0].astype(np.int64) | (xt[..., 1].astype(np.int64) << 16)
    bits = ((mask[..., :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(Hh_, NT, -1)[..., :B]
    return np.where(bits.astype(bool), tok, -1).reshape(Hh_, NT * B)


def full_attention(q, k, v, scale: float = 0.0):
    """Alg. 1 l.647-648: A_fu = softmax(Q K^T / sqrt(d)), O_fu = A_fu V per head on the
    untiled tokens (numpy fp64 matmul as the library step).  Returns O_fu [Hh, N, d]."""
    qd, kd, vd = (bf16_bits_to_f64(a) for a in (q, k, v))
    d = qd.shape[-1]
    sc = scale if scale > 0 else 1.0 / np.sqrt(d)
    out = np.empty_like(qd)
    for h in range(qd.shape[0]):
        l = (qd[h] @ kd[h].T) * sc
        l -= l.max(axis=1, keepdims=True)
        a = np.exp(l)
        a /= a.sum(axis=1, keepdims=True)
        out[h] = a @ vd[h]
    return out


def tiling_search_errors(q, k, v, lat, k_top: int, cands=None, o_fu=None, nthreads=None):
    """Alg. 1, Eq. 9, one calibration sample:
    for every candidate pi: tile Q, K, V with pi (l.652); oracle mask M~ = Top-k of the
    max-pooled full attention map (l.653-656; RowNorm is a positive per-row scale and does
    not change a row's Top-k, reading R20); O_sp = UnTile(SparseAttn(Q~, K~, V~, M~)) (l.658);
    E[h, pi] = ||O_fu - O_sp||_F^2 over the real tokens (l.659).
    k_top is clamped to N_T(pi) (R20).  Returns E [Hh, |cands|] fp64."""
    q = np.ascontiguousarray(q, dtype=np.uint16)
    Hh, N, d = q.shape
    cands = list(cands) if cands is not None else omega(128)
    if o_fu is None:
        o_fu = full_attention(q, k, v)
    E = np.zeros((Hh, len(cands)))
    for c, pi in enumerate(cands):
        qt, cnt, mask = tile_permute(q, lat, [pi])
        kt, _, _ = tile_permute(k, lat, [pi])
        vt, _, _ = tile_permute(v, lat, [pi])
        NT = qt.shape[1]
        s = target_scores(qt, kt, mask, nthreads=nthreads)
        idx = topk(s, min(k_top, NT))
        o_t = sparse_attn(qt, kt, vt, idx, mask, nthreads=nthreads)
        perm = token_index(lat, [pi], Hh)
        for h in range(Hh):
            real = perm[h] >= 0
            o_sp = np.empty((N, d))
            o_sp[perm[h][real]] = o_t[h].reshape(-1, d)[real]
            E[h, c] = ((o_fu[h] - o_sp) ** 2).sum()
    return E


def bf16_bits_to_f64(x: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (for pins written in numpy)."""
    return (np.asarray(x, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp64 -> bf16 bit patterns (via fp32; test helper)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r
