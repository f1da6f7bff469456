"""Head-aware tiling search on the GPU (Alg. 1; Eq. 8-9).

For each calibration sample and every candidate tiling pi in Omega (all (p_t, p_h, p_w)
with p_t p_h p_w = B), every head accumulates E[h, pi] += ||O_fu - O_sp(pi)||_F^2, where
O_sp(pi) is the tile-sparse attention under the ORACLE mask of pi (Top-k of the max-pooled
full attention map, Eq. 4) mapped back to token order.  pi*_h = argmin_pi E[h, pi].

Every step runs in libveda kernels (tiling, target scores, top-k, sparse attention,
untiling, squared error).  One dense attention pass per sample gives O_fu and the
per-token row lse; lse_u does not depend on the tiling, so it is re-tiled for each pi
(veda_tile_permute_scalar) instead of recomputing the full softmax |Omega| times as
Alg. 1 l.653 literally does -- same numbers, 1/|Omega| of the dense work.
Readings (R20): RowNorm is a positive per-row scale and does not change a row's
Top-k, so it is not applied; k_top is clamped to N_T(pi).
"""
from __future__ import annotations

import torch

from . import veda


def omega(B: int):
    """Eq. 8: (p_t, p_h, p_w) in N^3 with p_t p_h p_w = B, lexicographic.  libveda tiles
    need powers of two, which is every factorisation of B in {64, 128}."""
    return [(pt, ph, B // (pt * ph)) for pt in range(1, B + 1) if B % pt == 0
            for ph in range(1, B // pt + 1) if (B // pt) % ph == 0]


class TilingSearch:
    """Accumulates the error cube E over calibration samples.

    add_sample(q, k, v): bf16 [Hh, N, d] CUDA tensors of one layer's heads.
    errors(): E [Hh, |Omega|] fp64 (host); best(): pi* per head."""

    def __init__(self, lat, Hh: int, d: int, k_top: int, B: int = 128, cands=None, device="cuda"):
        self.lat, self.Hh, self.d, self.k_top = tuple(lat), Hh, d, int(k_top)
        self.cands = [tuple(c) for c in (cands if cands is not None else omega(B))]
        self.dev = torch.device(device)
        # [|Omega|, Hh] so that each candidate's row is a contiguous [Hh] vector for veda_sq_err
        self.err = torch.zeros((len(self.cands), Hh), dtype=torch.float64, device=self.dev)
        # reference tiling for the dense pass: the candidate with the fewest padded tiles
        self.ref = min(self.cands, key=lambda c: veda.tiled_shape(self.lat, [c], Hh).n_tiles)
        self.samples = 0

    def _tile3(self, q, k, v, cfg):
        qt, cnt, mask = veda.tile_permute(q, self.lat, [cfg])
        kt, _, _ = veda.tile_permute(k, self.lat, [cfg], meta=False)
        vt, _, _ = veda.tile_permute(v, self.lat, [cfg], meta=False)
        return qt, kt, vt, cnt, mask

    def full_attention(self, q, k, v):
        """O_fu [Hh, N, d] bf16 and the per-token row lse [Hh, N] fp32 (Alg. 1 l.647-648)."""
        qt, kt, vt, _, mask = self._tile3(q, k, v, self.ref)
        NT = qt.shape[1]
        dense = torch.arange(NT, dtype=torch.int32, device=self.dev).expand(self.Hh, NT, NT).contiguous()
        o_t, lse_t = veda.sparse_attn_fwd(qt, kt, vt, dense, mask, want_lse=True)
        return veda.tile_unpermute(o_t, self.lat, [self.ref]), veda.tile_unpermute_scalar(lse_t, self.lat, [self.ref])

    def candidate(self, q, k, v, lse_tok, cfg):
        """Oracle mask of one candidate and its sparse output in token order (Alg. 1 l.652-658)."""
        qt, kt, vt, _, mask = self._tile3(q, k, v, cfg)
        NT = qt.shape[1]
        lse_t = veda.tile_permute_scalar(lse_tok, self.lat, [cfg])
        s_tgt = veda.target_scores(qt, kt, mask, lse_t)
        idx = veda.select_topk(s_tgt, min(self.k_top, NT))
        o_t = veda.sparse_attn_fwd(qt, kt, vt, idx, mask)
        return veda.tile_unpermute(o_t, self.lat, [cfg]), idx

    def add_sample(self, q, k, v):
        o_fu, lse_tok = self.full_attention(q, k, v)
        for c, cfg in enumerate(self.cands):
            o_sp, _ = self.candidate(q, k, v, lse_tok, cfg)
            veda.sq_err(o_fu, o_sp, self.err[c])  # Alg. 1 l.659
        self.samples += 1

    def errors(self):
        return self.err.t().cpu()

    def best(self):
        """pi*_h = argmin over Omega of E[h, pi] (Alg. 1 l.666)."""
        e = self.errors()
        return [self.cands[int(j)] for j in e.argmin(dim=1)]
