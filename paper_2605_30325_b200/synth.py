"""Seeded synthetic inputs shaped like Wan2.1 / Waver video-DiT attention layers.

This module holds NONE of the method's arithmetic (no tiling, pooling, scoring,
top-k or attention).  It only draws inputs; both the CUDA path and the fp64
oracle consume what it returns.  Recipe (following
SURVEY.md §8(d) d3):

* Q_h, K_h = bf16(RoPE3D(alpha * u_h + sigma * eps)), alpha = 16, sigma = 1, with a
  unit vector u_h per head shared by Q and K and independent N(0,1) noise eps.
  RoPE3D uses the Wan2.1 head-dim split (d - 4*floor(d/6), 2*floor(d/6),
  2*floor(d/6)) for (t, h, w), theta = 10000, interleaved pairs, integer latent
  positions.  The paper's backbones use 3D RoPE.
* Head kinds cycle (PAPER.md:235-237 head diversity): u_h energy in all bands;
  temporal band only; spatial bands only.
* V ~ N(0, 1).
* Scorer weights: Xavier-uniform fp32, zero biases unless
  ``random_bias`` is set (tests use non-zero biases to exercise the bias path).
* Seeds: every tensor's seed is a hash of (master seed, preset name, GLOBAL head
  index, tensor id), so a head-sharded run regenerates exactly the data of the
  single-GPU run on the same device type.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import torch

MASTER_SEED = 20260517
ALPHA = 16.0
SIGMA = 1.0
THETA = 10000.0


@dataclass(frozen=True)
class Preset:
    name: str
    lat: tuple  # (T, H, W) latent grid
    heads: int
    d: int
    cfg: tuple  # (pt, ph, pw)
    sparsity: float


# BASELINE.json configs (tiny; Wan2.1-1.3B 480P/81f; Wan2.1-14B 720P/81f; Waver-12B 720P/241f)
PRESETS = {
    "tiny": Preset("tiny", (4, 8, 8), 1, 64, (4, 4, 4), 0.50),
    "wan1.3b": Preset("wan1.3b", (21, 30, 52), 12, 128, (4, 4, 8), 0.90),
    "wan14b": Preset("wan14b", (21, 45, 80), 40, 128, (4, 4, 8), 0.95),
    "waver12b": Preset("waver12b", (61, 45, 80), 24, 128, (4, 4, 8), 0.95),
}

# head-aware mode cycles the paper's static shapes per head
HEAD_AWARE_CFGS = ((4, 4, 8), (8, 4, 4), (4, 8, 4), (8, 8, 2))


def seed_of(*parts) -> int:
    h = hashlib.sha256(("/".join(str(p) for p in (MASTER_SEED,) + parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def _gen(device, *parts) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed_of(*parts))
    return g


def rope_split(d: int):
    f = d // 6
    return d - 4 * f, 2 * f, 2 * f


def _rope_angles(lat, d, device):
    """[N, d/2] rotation angles for interleaved pairs, Wan2.1 3D split."""
    T, H, W = lat
    dt, dh, dw = rope_split(d)
    t = torch.arange(T, device=device, dtype=torch.float32)
    h = torch.arange(H, device=device, dtype=torch.float32)
    w = torch.arange(W, device=device, dtype=torch.float32)

    def freqs(n):
        i = torch.arange(n // 2, device=device, dtype=torch.float32)
        return THETA ** (-2.0 * i / n)

    at = (t[:, None] * freqs(dt)[None, :])[:, None, None, :].expand(T, H, W, dt // 2)
    ah = (h[:, None] * freqs(dh)[None, :])[None, :, None, :].expand(T, H, W, dh // 2)
    aw = (w[:, None] * freqs(dw)[None, :])[None, None, :, :].expand(T, H, W, dw // 2)
    return torch.cat([at, ah, aw], dim=-1).reshape(T * H * W, d // 2)


def _apply_rope(x, ang):
    x0, x1 = x[..., 0::2], x[..., 1::2]
    c, s = torch.cos(ang), torch.sin(ang)
    out = torch.empty_like(x)
    out[..., 0::2] = x0 * c - x1 * s
    out[..., 1::2] = x0 * s + x1 * c
    return out


def _head_direction(preset_name, gh, d, device):
    g = _gen(device, preset_name, gh, "u")
    u = torch.randn(d, generator=g, device=device, dtype=torch.float32)
    dt, dh, dw = rope_split(d)
    kind = gh % 3
    if kind == 1:  # temporal band only
        u[dt:] = 0
    elif kind == 2:  # spatial bands only
        u[:dt] = 0
    return u / u.norm()


def qkv(preset: Preset | str, heads=None, device="cpu", layout="hnd", lat=None, d=None,
        alpha=ALPHA, sigma=SIGMA):
    """Return (q, k, v) bf16 tensors for the given GLOBAL head indices.

    layout "hnd" -> [Hh, N, d] contiguous; "nhd" -> [N, Hh, d] contiguous.
    ``lat``/``d`` override the preset's shape (tests use small toys).
    """
    if isinstance(preset, str):
        preset = PRESETS[preset]
    lat = tuple(lat) if lat is not None else preset.lat
    d = d if d is not None else preset.d
    if heads is None:
        heads = range(preset.heads)
    heads = list(heads)
    N = lat[0] * lat[1] * lat[2]
    ang = _rope_angles(lat, d, device)
    outs = {n: torch.empty((len(heads), N, d), dtype=torch.bfloat16, device=device) for n in "qkv"}
    for li, gh in enumerate(heads):
        u = _head_direction(preset.name, gh, d, device)
        for name in "qk":
            g = _gen(device, preset.name, lat, d, gh, name)
            eps = torch.randn((N, d), generator=g, device=device, dtype=torch.float32)
            x = alpha * u[None, :] + sigma * eps
            outs[name][li] = _apply_rope(x, ang).to(torch.bfloat16)
        g = _gen(device, preset.name, lat, d, gh, "v")
        outs["v"][li] = torch.randn((N, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    if layout == "nhd":
        return tuple(outs[n].transpose(0, 1).contiguous() for n in "qkv")
    return outs["q"], outs["k"], outs["v"]


def scorer_weights(preset: Preset | str, heads=None, d=None, d_hidden=None, d_lat=None,
                   random_bias=False, device="cpu"):
    """Xavier-uniform fp32 scorer weights, per global head.

    Returns dict with w1q,b1q,w2q,b2q,w1k,b1k,w2k,b2k: W1 [Hh,3d,dh], b1 [Hh,dh],
    W2 [Hh,dh,dl], b2 [Hh,dl].  Defaults (R8): dh = 2*3d, dl = d.
    """
    if isinstance(preset, str):
        preset = PRESETS[preset]
    d = d if d is not None else preset.d
    din = 3 * d
    dh = d_hidden if d_hidden is not None else 2 * din
    dl = d_lat if d_lat is not None else d
    if heads is None:
        heads = range(preset.heads)
    heads = list(heads)
    out = {}
    for side in "qk":
        w1 = torch.empty((len(heads), din, dh), dtype=torch.float32)
        w2 = torch.empty((len(heads), dh, dl), dtype=torch.float32)
        b1 = torch.zeros((len(heads), dh), dtype=torch.float32)
        b2 = torch.zeros((len(heads), dl), dtype=torch.float32)
        for li, gh in enumerate(heads):
            g = _gen("cpu", preset.name, d, dh, dl, gh, side, "w1")
            a1 = math.sqrt(6.0 / (din + dh))
            w1[li] = (torch.rand((din, dh), generator=g) * 2 - 1) * a1
            g = _gen("cpu", preset.name, d, dh, dl, gh, side, "w2")
            a2 = math.sqrt(6.0 / (dh + dl))
            w2[li] = (torch.rand((dh, dl), generator=g) * 2 - 1) * a2
            if random_bias:
                g = _gen("cpu", preset.name, d, dh, dl, gh, side, "b")
                b1[li] = torch.randn(dh, generator=g) * 0.1
                b2[li] = torch.randn(dl, generator=g) * 0.1
        out[f"w1{side}"], out[f"b1{side}"] = w1.to(device), b1.to(device)
        out[f"w2{side}"], out[f"b2{side}"] = w2.to(device), b2.to(device)
    return out


def random_index_lists(Hh, n_tiles, k, seed_parts=("R2",), device="cpu"):
    """Regime R2: uniformly random k-subsets per row, ascending."""
    g = _gen("cpu", *seed_parts, Hh, n_tiles, k)
    r = torch.rand((Hh, n_tiles, n_tiles), generator=g)
    # a uniformly random permutation prefix per row, then ascending
    idx = torch.argsort(r, dim=-1)[..., :k].sort(dim=-1).values.to(torch.int32)
    return idx.to(device)


def latent_tokens(lat) -> int:
    return lat[0] * lat[1] * lat[2]
