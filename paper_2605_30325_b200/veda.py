"""Python binding of libveda (include/veda.h): argument marshalling only.

Every step of the path runs in the CUDA kernels of libveda.so; this module only
checks tensor properties, allocates outputs with torch (device memory), and passes
raw pointers and the current CUDA stream through ctypes.  There is no CPU or
PyTorch fallback: if the library or a B200 is missing, calls raise.

Names follow the C ABI:  tile_permute, tile_score (trippool / project /
pair_scores), select_topk, sparse_attn_fwd, tile_unpermute, plus the composed
``sparse_attention`` (the five steps in order, Alg. 2 + Eq. 2).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VEDA_LIB", os.path.join(_HERE, "libveda.so"))

VEDA_STATUS = ["VEDA_OK", "VEDA_ERR_NULL", "VEDA_ERR_SHAPE", "VEDA_ERR_CONFIG", "VEDA_ERR_K_RANGE",
               "VEDA_ERR_ALIGN", "VEDA_ERR_WORKSPACE", "VEDA_ERR_INDEX", "VEDA_ERR_NONFINITE",
               "VEDA_ERR_CUDA", "VEDA_ERR_ARCH"]

EXPORTS = ["veda_tiled_shape_of", "veda_k_for_sparsity", "veda_tile_score_workspace", "veda_tile_permute",
           "veda_tile_score", "veda_select_topk", "veda_sparse_attn_fwd", "veda_tile_unpermute",
           "veda_trippool", "veda_project", "veda_pair_scores", "veda_status_str", "veda_last_error",
           "veda_launch_count", "veda_check_device", "veda_tile_permute_pool", "veda_tile_score_pooled",
           "veda_target_scores", "veda_tile_recall", "veda_tile_permute_scalar", "veda_tile_unpermute_scalar",
           "veda_sq_err", "veda_sparse_attention_host_workspace", "veda_sparse_attention_host",
           "veda_tile_pool", "veda_sparse_attn_fwd_tokens", "veda_sparse_attn_fwd_tokens_units",
           "veda_tile_pool_heads", "veda_validate_index", "veda_validate_finite", "veda_set_debug",
           "veda_tile_pool_local", "veda_sparse_attn_fwd_tokens_local", "veda_tile_select_workspace",
           "veda_tile_select_pooled", "veda_scorer_prepare_bytes", "veda_scorer_prepare", "veda_tile_pool_qk"]


class VedaError(RuntimeError):
    pass


class Latent(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32)]


class TileCfg(ctypes.Structure):
    _fields_ = [("pt", ctypes.c_int32), ("ph", ctypes.c_int32), ("pw", ctypes.c_int32)]


class TiledShape(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("hp", ctypes.c_int32), ("wp", ctypes.c_int32), ("B", ctypes.c_int32),
                ("n_tiles", ctypes.c_int32), ("reserved", ctypes.c_int32), ("n_pad", ctypes.c_int64)]


class Scorer(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int32), ("d_hidden", ctypes.c_int32), ("d_lat", ctypes.c_int32)] + [
        (n, ctypes.c_void_p) for n in ("w1q", "b1q", "w2q", "b2q", "w1k", "b1k", "w2k", "b2k", "prepared")]


_lib = None


def load(path: str = LIB_PATH):
    """Load libveda.so and declare signatures.  Raises if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise VedaError(f"{path} not built; run `python -m paper_2605_30325_b200.build`")
    lib = ctypes.CDLL(path)
    P, i32, i64, f32, f64, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                 ctypes.c_double, ctypes.c_size_t)
    sig = {
        "veda_tiled_shape_of": ([Latent, P, i32, P], i32),
        "veda_k_for_sparsity": ([i32, f64], i32),
        "veda_tile_score_workspace": ([i32, i32, i32, P, P], i32),
        "veda_tile_permute": ([P, i64, i64, Latent, P, i32, i32, P, P, P, P], i32),
        "veda_tile_permute_pool": ([P, i64, i64, Latent, P, i32, i32, P, P, P, P, P], i32),
        "veda_tile_score_pooled": ([P, P, P, i32, i32, i32, P, P, P, sz, P], i32),
        "veda_tile_select_workspace": ([i32, i32, i32, P, i32, P], i32),
        "veda_scorer_prepare_bytes": ([i32, i32, P, P], i32),
        "veda_scorer_prepare": ([i32, i32, P, P, sz, P], i32),
        "veda_tile_select_pooled": ([P, P, P, i32, i32, i32, P, i32, i32, P, P, sz, P], i32),
        "veda_tile_score": ([P, P, P, P, i32, i32, i32, i32, P, P, P, sz, P], i32),
        "veda_select_topk": ([P, i32, i32, i32, P, P], i32),
        "veda_sparse_attn_fwd": ([P, P, P, P, P, i32, i32, i32, i32, i32, f32, P, P, P], i32),
        "veda_tile_unpermute": ([P, Latent, P, i32, i32, P, i64, i64, P], i32),
        "veda_trippool": ([P, P, i32, i32, i32, i32, P, P], i32),
        "veda_project": ([P, i32, i32, i32, i32, i32, P, P, P, P, P, P, P], i32),
        "veda_pair_scores": ([P, P, P, i32, i32, i32, P, P], i32),
        "veda_target_scores": ([P, P, P, P, i32, i32, i32, i32, f32, P, P], i32),
        "veda_tile_recall": ([P, P, P, i64, i32, i32, P, P], i32),
        "veda_tile_permute_scalar": ([P, i64, Latent, P, i32, f32, P, P], i32),
        "veda_tile_unpermute_scalar": ([P, Latent, P, i32, P, i64, P], i32),
        "veda_sq_err": ([P, P, i64, i64, i32, P, P], i32),
        "veda_sparse_attention_host_workspace": ([Latent, P, i32, i32, i32, P, i32, P], i32),
        "veda_sparse_attention_host": ([P, P, P, i64, i64, Latent, P, i32, i32, i32, P, i32, P, P, sz, P], i32),
        "veda_tile_pool": ([P, i64, i64, Latent, P, i32, i32, P, P, P, P], i32),
        "veda_tile_pool_qk": ([P, P, i64, i64, Latent, P, i32, i32, P, P, P, P, P], i32),
        "veda_tile_pool_heads": ([P, i64, i64, Latent, P, i32, i32, i32, i32, P, P, P, P], i32),
        "veda_sparse_attn_fwd_tokens": ([P, P, P, i64, i64, Latent, P, i32, i32, P, P, i32, f32, P, i64, i64, P, P],
                                        i32),
        "veda_sparse_attn_fwd_tokens_units": ([P, P, P, i64, i64, Latent, P, i32, i32, P, P, i32, f32, P, i64, i64, P,
                                               i32, i32, P], i32),
        "veda_status_str": ([i32], ctypes.c_char_p),
        "veda_last_error": ([], ctypes.c_char_p),
        "veda_launch_count": ([], ctypes.c_uint64),
        "veda_check_device": ([], i32),
        "veda_validate_index": ([P, i64, i32, i32, P, P], i32),
        "veda_validate_finite": ([P, i64, i64, i32, i64, i32, P, P], i32),
        "veda_set_debug": ([i32], i32),
        "veda_tile_pool_local": ([P, i64, i64, Latent, P, i32, i32, i32, i32, P, P, P, P], i32),
        "veda_sparse_attn_fwd_tokens_local": ([P, P, P, i64, i64, Latent, P, i32, i32, i32, i32, P, P, i32, f32, P,
                                               i64, i64, P, P], i32),
    }
    for name, (args, res) in sig.items():
        if path != os.path.join(_HERE, "libveda.so") and not hasattr(lib, name):
            continue  # an older library under VEDA_LIB (A/B timing): newer entry points absent
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(st: int, what: str):
    if st != 0:
        lib = load()
        raise VedaError(f"{what}: {VEDA_STATUS[st] if st < len(VEDA_STATUS) else st}: "
                        f"{lib.veda_last_error().decode()}")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _cfg_array(cfgs, Hh):
    cfgs = [tuple(c) for c in cfgs]
    if len(cfgs) == 1 and Hh > 1:
        cfgs = cfgs * Hh
    if len(cfgs) != Hh:
        raise VedaError(f"{len(cfgs)} tile configs for {Hh} heads")
    arr = (TileCfg * Hh)(*[TileCfg(*c) for c in cfgs])
    return arr


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise VedaError("libveda takes CUDA tensors (no CPU fallback)")


def launch_count() -> int:
    return int(load().veda_launch_count())


def check_device():
    _check(load().veda_check_device(), "check_device")


FLAG_INDEX_RANGE, FLAG_INDEX_ORDER, FLAG_NONFINITE = 1, 2, 4


def set_debug(on: bool) -> bool:
    """Debug mode (include/veda.h): entry points validate their inputs and return
    VEDA_ERR_INDEX / VEDA_ERR_NONFINITE.  Returns the previous setting."""
    return bool(load().veda_set_debug(1 if on else 0))


def validate_index(idx: torch.Tensor, n_tiles: int) -> int:
    """VEDA_FLAG_* bits for kept-tile lists idx [..., k] (synchronises the current stream)."""
    _need_cuda(idx)
    k = idx.shape[-1]
    flags = torch.zeros(1, dtype=torch.int32, device=idx.device)
    _check(load().veda_validate_index(_ptr(idx), idx.numel() // k, n_tiles, k, _ptr(flags), _stream()),
           "validate_index")
    return int(flags.item())


def validate_finite(x: torch.Tensor) -> int:
    """VEDA_FLAG_NONFINITE if the bf16 tensor [Hh, N, d] (any strides, d contiguous) holds Inf/NaN."""
    _need_cuda(x)
    Hh, n, d = x.shape
    flags = torch.zeros(1, dtype=torch.int32, device=x.device)
    _check(load().veda_validate_finite(_ptr(x), x.stride(0), x.stride(1), Hh, n, d, _ptr(flags), _stream()),
           "validate_finite")
    return int(flags.item())


@dataclass
class TiledShapeInfo:
    tp: int
    hp: int
    wp: int
    B: int
    n_tiles: int
    n_pad: int


def tiled_shape(lat, cfgs, Hh: int) -> TiledShapeInfo:
    out = TiledShape()
    arr = _cfg_array(cfgs, Hh)
    _check(load().veda_tiled_shape_of(Latent(*lat), arr, Hh, ctypes.byref(out)), "tiled_shape_of")
    return TiledShapeInfo(out.tp, out.hp, out.wp, out.B, out.n_tiles, out.n_pad)


def k_for_sparsity(n_tiles: int, sparsity: float) -> int:
    return int(load().veda_k_for_sparsity(n_tiles, float(sparsity)))


def tile_permute(x: torch.Tensor, lat, cfgs, out=None, meta=True):
    """x: bf16 [Hh, N, d] view (last stride 1; e.g. x_nhd.transpose(0,1)).
    Returns (x_tiled [Hh,N_T,B,d], tile_count [Hh,N_T] int32 | None, slot_mask [Hh,N_T,B/32] | None)."""
    _need_cuda(x)
    assert x.dtype == torch.bfloat16 and x.dim() == 3 and x.stride(2) == 1
    Hh, N, d = x.shape
    sh = tiled_shape(lat, cfgs, Hh)
    if out is None:
        out = torch.empty((Hh, sh.n_tiles, sh.B, d), dtype=torch.bfloat16, device=x.device)
    cnt = mask = None
    if meta:
        cnt = torch.empty((Hh, sh.n_tiles), dtype=torch.int32, device=x.device)
        mask = torch.empty((Hh, sh.n_tiles, sh.B // 32), dtype=torch.int32, device=x.device)
    st = load().veda_tile_permute(_ptr(x), x.stride(0), x.stride(1), Latent(*lat), _cfg_array(cfgs, Hh), Hh, d,
                                  _ptr(out), _ptr(cnt), _ptr(mask), _stream())
    _check(st, "tile_permute")
    return out, cnt, mask


def tile_permute_pool(x: torch.Tensor, lat, cfgs, out=None):
    """Fused tiling + TripPool (one HBM pass): returns (x_tiled, tile_count, slot_mask, z)."""
    _need_cuda(x)
    assert x.dtype == torch.bfloat16 and x.dim() == 3 and x.stride(2) == 1
    Hh, N, d = x.shape
    sh = tiled_shape(lat, cfgs, Hh)
    if out is None:
        out = torch.empty((Hh, sh.n_tiles, sh.B, d), dtype=torch.bfloat16, device=x.device)
    cnt = torch.empty((Hh, sh.n_tiles), dtype=torch.int32, device=x.device)
    mask = torch.empty((Hh, sh.n_tiles, sh.B // 32), dtype=torch.int32, device=x.device)
    z = torch.empty((Hh, sh.n_tiles, 3 * d), dtype=torch.float32, device=x.device)
    st = load().veda_tile_permute_pool(_ptr(x), x.stride(0), x.stride(1), Latent(*lat), _cfg_array(cfgs, Hh), Hh, d,
                                       _ptr(out), _ptr(cnt), _ptr(mask), _ptr(z), _stream())
    _check(st, "tile_permute_pool")
    return out, cnt, mask, z


def tile_unpermute(o_tiled: torch.Tensor, lat, cfgs, out=None):
    """o_tiled [Hh,N_T,B,d] -> out [Hh, N, d] (or into a given [Hh,N,d] view)."""
    _need_cuda(o_tiled)
    Hh, NT, B, d = o_tiled.shape
    N = lat[0] * lat[1] * lat[2]
    if out is None:
        out = torch.empty((Hh, N, d), dtype=torch.bfloat16, device=o_tiled.device)
    assert out.stride(2) == 1
    st = load().veda_tile_unpermute(_ptr(o_tiled), Latent(*lat), _cfg_array(cfgs, Hh), Hh, d, _ptr(out),
                                    out.stride(0), out.stride(1), _stream())
    _check(st, "tile_unpermute")
    return out


def tile_permute_scalar(x: torch.Tensor, lat, cfgs, pad: float = 0.0, out=None):
    """Per-token fp32 x [Hh, N] (last stride 1) -> [Hh, N_T, B] in the tiling of cfgs."""
    _need_cuda(x)
    Hh = x.shape[0]
    sh = tiled_shape(lat, cfgs, Hh)
    if out is None:
        out = torch.empty((Hh, sh.n_tiles, sh.B), dtype=torch.float32, device=x.device)
    assert x.dtype == torch.float32 and x.stride(-1) == 1
    st = load().veda_tile_permute_scalar(_ptr(x), x.stride(0), Latent(*lat), _cfg_array(cfgs, Hh), Hh, float(pad),
                                         _ptr(out), _stream())
    _check(st, "tile_permute_scalar")
    return out


def tile_unpermute_scalar(x_tiled: torch.Tensor, lat, cfgs, out=None):
    """[Hh, N_T, B] fp32 -> per-token [Hh, N] (padded slots dropped)."""
    _need_cuda(x_tiled)
    Hh = x_tiled.shape[0]
    N = lat[0] * lat[1] * lat[2]
    if out is None:
        out = torch.empty((Hh, N), dtype=torch.float32, device=x_tiled.device)
    st = load().veda_tile_unpermute_scalar(_ptr(x_tiled), Latent(*lat), _cfg_array(cfgs, Hh), Hh, _ptr(out),
                                           out.stride(0), _stream())
    _check(st, "tile_unpermute_scalar")
    return out


def sq_err(a: torch.Tensor, b: torch.Tensor, err: torch.Tensor):
    """err[h] += ||a[h] - b[h]||_F^2 for bf16 [Hh, ...] tensors (contiguous); err fp64 [Hh]."""
    _need_cuda(a, b, err)
    assert a.shape == b.shape and a.is_contiguous() and b.is_contiguous() and err.dtype == torch.float64
    Hh = a.shape[0]
    n = a[0].numel()
    st = load().veda_sq_err(_ptr(a), _ptr(b), n, n, Hh, _ptr(err), _stream())
    _check(st, "sq_err")
    return err


def trippool(x_tiled: torch.Tensor, slot_mask: torch.Tensor):
    _need_cuda(x_tiled, slot_mask)
    Hh, NT, B, d = x_tiled.shape
    z = torch.empty((Hh, NT, 3 * d), dtype=torch.float32, device=x_tiled.device)
    _check(load().veda_trippool(_ptr(x_tiled), _ptr(slot_mask), Hh, NT, B, d, _ptr(z), _stream()), "trippool")
    return z


def project(z: torch.Tensor, w1, b1, w2, b2):
    _need_cuda(z, w1, b1, w2, b2)
    Hh, NT, din = z.shape
    dh, dl = w1.shape[-1], w2.shape[-1]
    hid = torch.empty((Hh, NT, dh), dtype=torch.float64, device=z.device)
    e = torch.empty((Hh, NT, dl), dtype=torch.float64, device=z.device)
    st = load().veda_project(_ptr(z), Hh, NT, din, dh, dl, _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2), _ptr(hid),
                             _ptr(e), _stream())
    _check(st, "project")
    return e


def pair_scores(eq: torch.Tensor, ek: torch.Tensor, tile_count: torch.Tensor):
    _need_cuda(eq, ek, tile_count)
    Hh, NT, dl = eq.shape
    s = torch.empty((Hh, NT, NT), dtype=torch.float32, device=eq.device)
    st = load().veda_pair_scores(_ptr(eq), _ptr(ek), _ptr(tile_count), Hh, NT, dl, _ptr(s), _stream())
    _check(st, "pair_scores")
    return s


def make_scorer(w: dict):
    """ctypes veda_scorer from a dict of CUDA fp32 tensors (synth.scorer_weights layout)."""
    _need_cuda(*w.values())
    for v in w.values():
        assert v.dtype == torch.float32 and v.is_contiguous()
    din, dh = w["w1q"].shape[-2:]
    dl = w["w2q"].shape[-1]
    sc = Scorer(din, dh, dl, *[w[n].data_ptr() for n in ("w1q", "b1q", "w2q", "b2q", "w1k", "b1k", "w2k", "b2k")])
    return sc


def prepare_scorer(scorer: Scorer, Hh: int, d: int, device):
    """Fill a device buffer with the scorer's weight digit images (veda_scorer_prepare) and
    point ``scorer.prepared`` at it; returns the buffer (keep it alive with the scorer)."""
    n = ctypes.c_size_t(0)
    lib = load()
    _check(lib.veda_scorer_prepare_bytes(Hh, d, ctypes.byref(scorer), ctypes.byref(n)), "scorer_prepare_bytes")
    buf = torch.empty(n.value, dtype=torch.uint8, device=device)
    scorer.prepared = None
    _check(lib.veda_scorer_prepare(Hh, d, ctypes.byref(scorer), _ptr(buf), n.value, _stream()), "scorer_prepare")
    torch.cuda.current_stream(device).synchronize()  # one-time setup: ready for calls on any stream
    scorer.prepared = buf.data_ptr()
    return buf


class ScoreWorkspace:
    """Caller-owned workspace for tile_score, sized by veda_tile_score_workspace."""

    def __init__(self, Hh, n_tiles, d, scorer: Scorer, device):
        n = ctypes.c_size_t(0)
        _check(load().veda_tile_score_workspace(Hh, n_tiles, d, ctypes.byref(scorer), ctypes.byref(n)),
               "tile_score_workspace")
        self.nbytes = n.value
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)


def tile_score(q_tiled, k_tiled, tile_count, slot_mask, scorer: Scorer, workspace: ScoreWorkspace = None,
               out=None):
    _need_cuda(q_tiled, k_tiled, tile_count, slot_mask)
    Hh, NT, B, d = q_tiled.shape
    if workspace is None:
        workspace = ScoreWorkspace(Hh, NT, d, scorer, q_tiled.device)
    if out is None:
        out = torch.empty((Hh, NT, NT), dtype=torch.float32, device=q_tiled.device)
    st = load().veda_tile_score(_ptr(q_tiled), _ptr(k_tiled), _ptr(tile_count), _ptr(slot_mask), Hh, NT, B, d,
                                ctypes.byref(scorer), _ptr(out), _ptr(workspace.buf), workspace.nbytes, _stream())
    _check(st, "tile_score")
    return out


def tile_score_pooled(zq, zk, tile_count, scorer: Scorer, workspace: ScoreWorkspace = None, out=None):
    _need_cuda(zq, zk, tile_count)
    Hh, NT, din = zq.shape
    d = din // 3
    if workspace is None:
        workspace = ScoreWorkspace(Hh, NT, d, scorer, zq.device)
    if out is None:
        out = torch.empty((Hh, NT, NT), dtype=torch.float32, device=zq.device)
    st = load().veda_tile_score_pooled(_ptr(zq), _ptr(zk), _ptr(tile_count), Hh, NT, d, ctypes.byref(scorer),
                                       _ptr(out), _ptr(workspace.buf), workspace.nbytes, _stream())
    _check(st, "tile_score_pooled")
    return out


def select_chunk_heads(Hh: int, n_tiles: int, heads_per_chunk: int = 0) -> int:
    """Heads per score chunk of veda_tile_select_pooled (mirrors the library: as many heads
    as fit 128 MB of fp32 scores, at least one, unless given)."""
    if heads_per_chunk > 0:
        return min(heads_per_chunk, Hh)
    return max(1, min(Hh, (128 << 20) // (n_tiles * n_tiles * 4)))


class SelectWorkspace:
    """Caller-owned workspace for tile_select_pooled (score + top-k without a full S)."""

    def __init__(self, Hh, n_tiles, d, scorer: Scorer, device, heads_per_chunk=0):
        n = ctypes.c_size_t(0)
        _check(load().veda_tile_select_workspace(Hh, n_tiles, d, ctypes.byref(scorer), heads_per_chunk,
                                                 ctypes.byref(n)), "tile_select_workspace")
        self.nbytes = n.value
        self.heads_per_chunk = heads_per_chunk
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)


def tile_select_pooled(zq, zk, tile_count, scorer: Scorer, k: int, heads_per_chunk: int = 0,
                       workspace: SelectWorkspace = None, out=None):
    """Kept-tile lists [Hh, N_T, k] from pooled descriptors (phi, S_pred per head chunk, top-k)."""
    _need_cuda(zq, zk, tile_count)
    Hh, NT, din = zq.shape
    d = din // 3
    if workspace is None:
        workspace = SelectWorkspace(Hh, NT, d, scorer, zq.device, heads_per_chunk)
    if out is None:
        out = torch.empty((Hh, NT, k), dtype=torch.int32, device=zq.device)
    st = load().veda_tile_select_pooled(_ptr(zq), _ptr(zk), _ptr(tile_count), Hh, NT, d, ctypes.byref(scorer), k,
                                        workspace.heads_per_chunk, _ptr(out), _ptr(workspace.buf), workspace.nbytes,
                                        _stream())
    _check(st, "tile_select_pooled")
    return out


def select_topk(scores: torch.Tensor, k: int, out=None):
    _need_cuda(scores)
    Hh, NT, _ = scores.shape
    if out is None:
        out = torch.empty((Hh, NT, k), dtype=torch.int32, device=scores.device)
    _check(load().veda_select_topk(_ptr(scores), Hh, NT, k, _ptr(out), _stream()), "select_topk")
    return out


def sparse_attn_fwd(q_tiled, k_tiled, v_tiled, idx, slot_mask, scale: float = 0.0, out=None, want_lse=False):
    _need_cuda(q_tiled, k_tiled, v_tiled, idx, slot_mask)
    Hh, NT, B, d = q_tiled.shape
    k = idx.shape[-1]
    if out is None:
        out = torch.empty_like(q_tiled)
    lse = torch.empty((Hh, NT, B), dtype=torch.float32, device=q_tiled.device) if want_lse else None
    st = load().veda_sparse_attn_fwd(_ptr(q_tiled), _ptr(k_tiled), _ptr(v_tiled), _ptr(idx), _ptr(slot_mask), Hh,
                                     NT, B, d, k, float(scale), _ptr(out), _ptr(lse), _stream())
    _check(st, "sparse_attn_fwd")
    return (out, lse) if want_lse else out


def tile_pool_qk(q: torch.Tensor, k: torch.Tensor, lat, cfgs):
    """TripPool of Q and K in one launch (veda_tile_pool_qk).  Returns (zq, zk, tile_count,
    slot_mask)."""
    _need_cuda(q, k)
    assert q.dtype == torch.bfloat16 and q.stride() == k.stride() and q.shape == k.shape and q.stride(2) == 1
    Hh, N, d = q.shape
    sh = tiled_shape(lat, cfgs, Hh)
    zq = torch.empty((Hh, sh.n_tiles, 3 * d), dtype=torch.float32, device=q.device)
    zk = torch.empty_like(zq)
    cnt = torch.empty((Hh, sh.n_tiles), dtype=torch.int32, device=q.device)
    mask = torch.empty((Hh, sh.n_tiles, sh.B // 32), dtype=torch.int32, device=q.device)
    _check(load().veda_tile_pool_qk(_ptr(q), _ptr(k), q.stride(0), q.stride(1), Latent(*lat), _cfg_array(cfgs, Hh),
                                    Hh, d, _ptr(zq), _ptr(zk), _ptr(cnt), _ptr(mask), _stream()), "tile_pool_qk")
    return zq, zk, cnt, mask


def tile_pool(x: torch.Tensor, lat, cfgs, z=None, meta=True):
    """TripPool of every tile of x [Hh, N, d] read straight from token order (veda_tile_pool).
    Returns (z [Hh, N_T, 3d] fp32, tile_count | None, slot_mask | None)."""
    _need_cuda(x)
    assert x.dtype == torch.bfloat16 and x.dim() == 3 and x.stride(2) == 1
    Hh, N, d = x.shape
    sh = tiled_shape(lat, cfgs, Hh)
    if z is None:
        z = torch.empty((Hh, sh.n_tiles, 3 * d), dtype=torch.float32, device=x.device)
    cnt = mask = None
    if meta:
        cnt = torch.empty((Hh, sh.n_tiles), dtype=torch.int32, device=x.device)
        mask = torch.empty((Hh, sh.n_tiles, sh.B // 32), dtype=torch.int32, device=x.device)
    _check(load().veda_tile_pool(_ptr(x), x.stride(0), x.stride(1), Latent(*lat), _cfg_array(cfgs, Hh), Hh, d,
                                 _ptr(z), _ptr(cnt), _ptr(mask), _stream()), "tile_pool")
    return z, cnt, mask


def sparse_attn_fwd_tokens(q, k, v, lat, cfgs, idx, slot_mask, scale: float = 0.0, out=None, want_lse=False,
                           units=None):
    """Attention + untiling straight on token tensors [Hh, N, d] (veda_sparse_attn_fwd_tokens).
    Rows of padded slots are not written, so ``out`` (default: zeros) keeps its values there.
    ``units=(begin, end)`` computes only that range of the flattened (head, query tile) space
    (veda_sparse_attn_fwd_tokens_units); rows outside it are not written either."""
    _need_cuda(q, k, v, idx, slot_mask)
    Hh, N, d = q.shape
    if not (k.stride() == q.stride() and v.stride() == q.stride()):
        raise VedaError("sparse_attn_fwd_tokens: q, k, v must share strides")
    NT, kk = idx.shape[1], idx.shape[2]
    B = slot_mask.shape[2] * 32
    if out is None:
        out = torch.zeros((Hh, N, d), dtype=torch.bfloat16, device=q.device)
    lse = torch.empty((Hh, NT, B), dtype=torch.float32, device=q.device) if want_lse else None
    args = (_ptr(q), _ptr(k), _ptr(v), q.stride(0), q.stride(1), Latent(*lat), _cfg_array(cfgs, Hh), Hh, d,
            _ptr(idx), _ptr(slot_mask), kk, float(scale), _ptr(out), out.stride(0), out.stride(1), _ptr(lse))
    if units is None:
        st = load().veda_sparse_attn_fwd_tokens(*args, _stream())
    else:
        st = load().veda_sparse_attn_fwd_tokens_units(*args, int(units[0]), int(units[1]), _stream())
    _check(st, "sparse_attn_fwd_tokens")
    return (out, lse) if want_lse else out


def target_scores(q_tiled, k_tiled, slot_mask, lse, scale: float = 0.0, out=None):
    """Eq. 4 pass 2: S_tgt [Hh, N_T, N_T] fp32 from the dense lse (see oracle_tile_mask)."""
    _need_cuda(q_tiled, k_tiled, slot_mask, lse)
    Hh, NT, B, d = q_tiled.shape
    if out is None:
        out = torch.empty((Hh, NT, NT), dtype=torch.float32, device=q_tiled.device)
    st = load().veda_target_scores(_ptr(q_tiled), _ptr(k_tiled), _ptr(slot_mask), _ptr(lse), Hh, NT, B, d,
                                   float(scale), _ptr(out), _stream())
    _check(st, "target_scores")
    return out


def oracle_tile_mask(q_tiled, k_tiled, v_tiled, slot_mask, k: int, scale: float = 0.0):
    """The oracle mask M~* of Eq. 4 / Alg. 3, both passes on the GPU:
    pass 1 = dense veda_sparse_attn_fwd (k = N_T) for the row lse, pass 2 =
    veda_target_scores, then veda_select_topk.  Returns (idx [Hh,N_T,k], S_tgt)."""
    Hh, NT, B, d = q_tiled.shape
    dense = torch.arange(NT, dtype=torch.int32, device=q_tiled.device).expand(Hh, NT, NT).contiguous()
    _, lse = sparse_attn_fwd(q_tiled, k_tiled, v_tiled, dense, slot_mask, scale=scale, want_lse=True)
    s_tgt = target_scores(q_tiled, k_tiled, slot_mask, lse, scale=scale)
    return select_topk(s_tgt, k), s_tgt


def tile_recall(idx_sp, idx_fu, tile_count=None, n_tiles=None, out=None):
    """Eq. 3 Recall@k (device fp64 scalar tensor).  idx [..., k]; n_tiles defaults to
    idx_sp.shape[-2] (square [Hh, N_T, k] lists)."""
    _need_cuda(idx_sp, idx_fu)
    k = idx_sp.shape[-1]
    NT = int(n_tiles) if n_tiles is not None else idx_sp.shape[-2]
    rows = idx_sp.numel() // k
    if out is None:
        out = torch.empty((), dtype=torch.float64, device=idx_sp.device)
    st = load().veda_tile_recall(_ptr(idx_sp), _ptr(idx_fu), _ptr(tile_count), rows, NT, k, _ptr(out), _stream())
    _check(st, "tile_recall")
    return out


class SparseAttention:
    """The whole hot path with preallocated buffers (one DiT attention layer call).

    q, k, v: bf16 [Hh, N, d] views on the GPU (any head / token strides shared by the
    three).  Steps (Alg. 2 + Eq. 2):

    * ``mode="tokens"`` (default): tile_pool Q/K (TripPool read
      straight from token order) -> tile_select_pooled (phi, S_pred and top-k per chunk of
      heads: no [Hh, N_T, N_T] score tensor) -> sparse_attn_fwd_tokens (tiles TMA'd from
      token order, rows stored to token order); no tiled copy of Q, K, V or O exists.
      ``keep_scores=True`` runs tile_score_pooled -> select_topk instead and keeps S in
      ``self.scores`` (parity tests; the lists are bit-identical);
    * ``mode="tiled"``: permute Q/K/V -> tile_score -> select_topk -> sparse_attn_fwd ->
      unpermute (the five-call form of include/veda.h; bit-identical output).
    """

    STEPS = {"tokens": ("pool", "score_topk", "attn", "untile"),
             "tokens_keep": ("pool", "score", "topk", "attn", "untile"),
             "tiled": ("permute", "score", "topk", "attn", "unpermute")}

    def __init__(self, lat, cfgs, Hh, d, scorer_weights: dict, sparsity=None, k=None, device="cuda",
                 mode="tokens", units=None, head_range=None, keep_scores=False):
        """``units=(begin, end)`` (tokens mode): a rank's share under shard.unit_range of the
        flattened (head, query tile) units of this Hh-head call.  Pooling (on the call's
        padded grid, veda_tile_pool_heads), scoring and top-k then run for the heads the
        share touches only, and the attention for the share's units only
        (veda_sparse_attn_fwd_tokens_units); q, k, v, out stay the whole call's tensors and
        only the share's output rows are written.

        ``head_range=range(h0, h1)`` (tokens mode): this object computes the heads [h0, h1)
        of an Hh-head call whose tile configs are ``cfgs`` (all Hh of them, so the padded
        grid, N_T and k are the whole call's -- a head subset's own grid can differ with
        head-aware tiling), but q, k, v, out and scorer_weights hold ONLY those heads
        ([h1 - h0, N, d]; the Ulysses front end's head shards).  Outputs are bit-identical
        to the same heads of the whole call."""
        if mode not in ("tokens", "tiled"):
            raise VedaError("mode must be one of ['tokens', 'tiled']")
        self.keep_scores = bool(keep_scores) or mode == "tiled"
        self.steps = self.STEPS["tiled" if mode == "tiled" else ("tokens_keep" if self.keep_scores else "tokens")]
        if (units is not None or head_range is not None) and mode != "tokens":
            raise VedaError("units / head_range: tokens mode only")
        if units is not None and head_range is not None:
            raise VedaError("units and head_range are exclusive")
        self.head_range = None
        if head_range is not None:
            if not (0 <= head_range.start <= head_range.stop <= Hh):
                raise VedaError(f"head_range {head_range} outside [0, {Hh}]")
            self.head_range = head_range
            NT0 = tiled_shape(lat, cfgs, Hh).n_tiles
            units = (head_range.start * NT0, head_range.stop * NT0)
        self.units = None if units is None else (int(units[0]), int(units[1]))
        self.lat, self.cfgs, self.Hh, self.d, self.mode = tuple(lat), list(cfgs), Hh, d, mode
        self.shape = tiled_shape(lat, cfgs, Hh)
        NT, B = self.shape.n_tiles, self.shape.B
        self.k = k if k is not None else k_for_sparsity(NT, sparsity)
        self.weights = scorer_weights
        self.scorer = make_scorer(scorer_weights)
        dev = torch.device(device)
        self.device = dev
        Hb = Hh if self.head_range is None else len(self.head_range)  # heads the buffers hold
        if mode == "tiled":
            mk = lambda: torch.empty((Hh, NT, B, d), dtype=torch.bfloat16, device=dev)
            self.qt, self.kt, self.vt, self.ot = mk(), mk(), mk(), mk()
        else:
            self.zq = torch.empty((Hb, NT, 3 * d), dtype=torch.float32, device=dev)
            self.zk = torch.empty((Hb, NT, 3 * d), dtype=torch.float32, device=dev)
        self.cnt = torch.empty((Hb, NT), dtype=torch.int32, device=dev)
        self.mask = torch.empty((Hb, NT, B // 32), dtype=torch.int32, device=dev)
        self.scores = torch.empty((Hb, NT, NT), dtype=torch.float32, device=dev) if self.keep_scores else None
        self.idx = torch.empty((Hb, NT, self.k), dtype=torch.int32, device=dev)
        self.heads = range(Hh)
        if self.head_range is not None:
            self.heads = self.head_range
            if len(self.heads):
                self.scorer = make_scorer(scorer_weights)
        elif self.units is not None:
            from .shard import heads_of_units

            if not (0 <= self.units[0] <= self.units[1] <= Hh * NT):
                raise VedaError(f"units {self.units} outside [0, {Hh * NT}]")
            self.heads = heads_of_units(range(*self.units), NT)
            h0, h1 = self.heads.start, self.heads.stop
            self.w_sub = {n: t[h0:h1] for n, t in scorer_weights.items()}
            if h1 > h0:
                self.scorer = make_scorer(self.w_sub)
        # W1 / W2 digit images once per object (static weights): no weight splits per call
        self._prep_buf = prepare_scorer(self.scorer, len(self.heads), d, dev) if len(self.heads) else None
        if self.keep_scores:
            self.ws = ScoreWorkspace(max(1, len(self.heads)), NT, d, self.scorer, dev)
        else:
            self.ws = SelectWorkspace(max(1, len(self.heads)), NT, d, self.scorer, dev)

    def tiled(self, q, k, v):
        """Tiled copies (q~, k~, v~) of the inputs (for the oracle-mask / target tools)."""
        lat, cfgs = self.lat, self.cfgs
        return (tile_permute(q, lat, cfgs, meta=False)[0], tile_permute(k, lat, cfgs, meta=False)[0],
                tile_permute(v, lat, cfgs, meta=False)[0])

    def capture(self, q, k, v, out):
        """Record one call on (q, k, v, out) into a CUDA graph and return it
        (``g.replay()`` re-runs every kernel of the call on those same buffers; the fused
        select's side-stream fork / join is captured with it).  Removes the per-call launch
        gaps: measured ~0.1 ms on the score + top-k step at Waver (tools/graph_bench.py).
        The library must already be warm on this device (one eager call first: the Phi
        table upload is synchronous)."""
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=q.device)
        s.wait_stream(torch.cuda.current_stream(q.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                self(q, k, v, out=out)
        torch.cuda.current_stream(q.device).wait_stream(s)
        return g

    def __call__(self, q, k, v, out=None, events=None):
        """Run the path; ``events`` (optional list of 6 torch.cuda.Event) brackets the steps."""
        lib, s = load(), _stream()
        Hh, d, lat = self.Hh, self.d, Latent(*self.lat)
        cfg = _cfg_array(self.cfgs, Hh)
        NT, B = self.shape.n_tiles, self.shape.B
        if out is None:
            Ho = Hh if self.head_range is None else len(self.head_range)
            out = torch.zeros((Ho, self.lat[0] * self.lat[1] * self.lat[2], d), dtype=torch.bfloat16,
                              device=q.device)
        ev = events or [None] * 6

        nmark = [0]

        def mark():  # events[i] after the i-th step (self.steps), events[0] at the start
            i = nmark[0]
            if i < len(ev) and ev[i] is not None:
                ev[i].record()
            nmark[0] += 1

        mark()
        if self.mode == "tokens":
            if not (k.stride() == q.stride() and v.stride() == q.stride()):
                raise VedaError("q, k, v must share strides")
            h0, h1 = self.heads.start, self.heads.stop
            if self.units is None:  # Q and K in one pooling launch
                _check(lib.veda_tile_pool_qk(_ptr(q), _ptr(k), q.stride(0), q.stride(1), lat, cfg, Hh, d,
                                             _ptr(self.zq), _ptr(self.zk), _ptr(self.cnt), _ptr(self.mask), s),
                       "tile_pool_qk")
            elif self.head_range is not None:  # head-shard tensors, the whole call's padded grid
                _check(lib.veda_tile_pool_local(_ptr(q), q.stride(0), q.stride(1), lat, cfg, Hh, d, h0, h1,
                                                _ptr(self.zq), _ptr(self.cnt), _ptr(self.mask), s), "tile_pool_local(q)")
                _check(lib.veda_tile_pool_local(_ptr(k), k.stride(0), k.stride(1), lat, cfg, Hh, d, h0, h1,
                                                _ptr(self.zk), None, None, s), "tile_pool_local(k)")
            else:  # the share's heads, on the whole call's padded grid
                _check(lib.veda_tile_pool_heads(_ptr(q), q.stride(0), q.stride(1), lat, cfg, Hh, d, h0, h1,
                                                _ptr(self.zq), _ptr(self.cnt), _ptr(self.mask), s), "tile_pool_heads(q)")
                _check(lib.veda_tile_pool_heads(_ptr(k), k.stride(0), k.stride(1), lat, cfg, Hh, d, h0, h1,
                                                _ptr(self.zk), None, None, s), "tile_pool_heads(k)")
            mark()
            # score / top-k buffers: the whole call's rows (units) or the shard's own (head_range)
            R = (lambda t, a, b: t[a:b]) if self.head_range is None else (lambda t, a, b: t)
            if self.keep_scores:
                if h1 > h0:
                    _check(lib.veda_tile_score_pooled(_ptr(R(self.zq, h0, h1)), _ptr(R(self.zk, h0, h1)),
                                                      _ptr(R(self.cnt, h0, h1)), h1 - h0, NT, d,
                                                      ctypes.byref(self.scorer), _ptr(R(self.scores, h0, h1)),
                                                      _ptr(self.ws.buf), self.ws.nbytes, s), "tile_score_pooled")
                mark()
                if h1 > h0:
                    _check(lib.veda_select_topk(_ptr(R(self.scores, h0, h1)), h1 - h0, NT, self.k,
                                                _ptr(R(self.idx, h0, h1)), s), "select_topk")
                mark()
            else:
                if h1 > h0:
                    _check(lib.veda_tile_select_pooled(_ptr(R(self.zq, h0, h1)), _ptr(R(self.zk, h0, h1)),
                                                       _ptr(R(self.cnt, h0, h1)), h1 - h0, NT, d,
                                                       ctypes.byref(self.scorer), self.k, self.ws.heads_per_chunk,
                                                       _ptr(R(self.idx, h0, h1)), _ptr(self.ws.buf), self.ws.nbytes,
                                                       s), "tile_select_pooled")
                mark()
            if self.units is None:
                _check(lib.veda_sparse_attn_fwd_tokens(_ptr(q), _ptr(k), _ptr(v), q.stride(0), q.stride(1), lat, cfg,
                                                       Hh, d, _ptr(self.idx), _ptr(self.mask), self.k, 0.0, _ptr(out),
                                                       out.stride(0), out.stride(1), None, s), "sparse_attn_fwd_tokens")
            elif self.head_range is not None:
                _check(lib.veda_sparse_attn_fwd_tokens_local(_ptr(q), _ptr(k), _ptr(v), q.stride(0), q.stride(1), lat,
                                                             cfg, Hh, d, h0, h1, _ptr(self.idx), _ptr(self.mask),
                                                             self.k, 0.0, _ptr(out), out.stride(0), out.stride(1),
                                                             None, s), "sparse_attn_fwd_tokens_local")
            else:
                _check(lib.veda_sparse_attn_fwd_tokens_units(_ptr(q), _ptr(k), _ptr(v), q.stride(0), q.stride(1), lat,
                                                             cfg, Hh, d, _ptr(self.idx), _ptr(self.mask), self.k, 0.0,
                                                             _ptr(out), out.stride(0), out.stride(1), None,
                                                             self.units[0], self.units[1], s),
                       "sparse_attn_fwd_tokens_units")
            mark()  # attn
            mark()  # untile (fused into the attention epilogue)
            return out
        # Q/K tiling and TripPool as two HBM-bound passes: measured faster than the fused
        # veda_tile_permute_pool (its extra registers halve the occupancy of the copy)
        _check(lib.veda_tile_permute(_ptr(q), q.stride(0), q.stride(1), lat, cfg, Hh, d, _ptr(self.qt),
                                     _ptr(self.cnt), _ptr(self.mask), s), "tile_permute(q)")
        _check(lib.veda_tile_permute(_ptr(k), k.stride(0), k.stride(1), lat, cfg, Hh, d, _ptr(self.kt), None, None,
                                     s), "tile_permute(k)")
        _check(lib.veda_tile_permute(_ptr(v), v.stride(0), v.stride(1), lat, cfg, Hh, d, _ptr(self.vt), None, None,
                                     s), "tile_permute(v)")
        mark()
        _check(lib.veda_tile_score(_ptr(self.qt), _ptr(self.kt), _ptr(self.cnt), _ptr(self.mask), Hh, NT, B, d,
                                   ctypes.byref(self.scorer), _ptr(self.scores), _ptr(self.ws.buf), self.ws.nbytes, s),
               "tile_score")
        mark()
        _check(lib.veda_select_topk(_ptr(self.scores), Hh, NT, self.k, _ptr(self.idx), s), "select_topk")
        mark()
        _check(lib.veda_sparse_attn_fwd(_ptr(self.qt), _ptr(self.kt), _ptr(self.vt), _ptr(self.idx), _ptr(self.mask),
                                        Hh, NT, B, d, self.k, 0.0, _ptr(self.ot), None, s), "sparse_attn_fwd")
        mark()
        _check(lib.veda_tile_unpermute(_ptr(self.ot), lat, cfg, Hh, d, _ptr(out), out.stride(0), out.stride(1), s),
               "tile_unpermute")
        mark()
        return out

    @property
    def LAUNCHES_PER_CALL(self):
        """Kernel launches of one call.  Scorer (INT8 Ozaki): phi = per side 2 x (split rows,
        split cols, GEMM) = 12, or 8 with prepared weights (no split cols: the object's
        default); the digit splits of e_q / e_k = 2; per chunk of heads the
        score GEMM + the top-k (one chunk with keep_scores: the full S, then select_topk).
        tokens: pool x2, scorer, attn;  tiled: permute x3, pool x2, scorer, attn, unpermute."""
        nh = max(1, len(self.heads))
        chunks = 1 if self.keep_scores else -(-nh // select_chunk_heads(nh, self.shape.n_tiles,
                                                                         self.ws.heads_per_chunk))
        scorer = (8 if self.scorer.prepared else 12) + 2 + 2 * chunks
        pool = 1 if self.units is None else 2  # Q and K in one launch on the whole-call path
        return {"tokens": pool + scorer + 1, "tiled": 3 + 2 + scorer + 1 + 1}

    def run_host(self, q, k, v, out=None, heads_per_chunk: int = 0):
        """The same call on HOST tensors (veda_sparse_attention_host): q, k, v, out are
        pinned CPU bf16 tensors, dense [Hh, N, d] or dense views [N, Hh, d] permuted to
        [Hh, N, d]; the library pipelines H2D / the five steps / D2H over head chunks.
        Returns ``out`` (valid once the current stream is synchronised)."""
        lib, s = load(), _stream()
        Hh, d = self.Hh, self.d
        N = self.lat[0] * self.lat[1] * self.lat[2]
        for t in (q, k, v):
            if t.is_cuda or t.dtype != torch.bfloat16 or tuple(t.shape) != (Hh, N, d):
                raise VedaError("run_host: q/k/v must be CPU bf16 [Hh, N, d]")
            if t.stride() != q.stride():
                raise VedaError("run_host: q/k/v must share one layout")
        if out is None:
            out = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, pin_memory=True)
        if out.stride() != q.stride():
            raise VedaError("run_host: out must have the layout of q")
        lat, cfg = Latent(*self.lat), _cfg_array(self.cfgs, Hh)
        key = (heads_per_chunk,)
        if getattr(self, "_host_ws_key", None) != key:
            nb = ctypes.c_size_t(0)
            _check(lib.veda_sparse_attention_host_workspace(lat, cfg, Hh, d, self.k, ctypes.byref(self.scorer),
                                                            heads_per_chunk, ctypes.byref(nb)),
                   "sparse_attention_host_workspace")
            self._host_ws = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
            self._host_ws_key = key
        _check(lib.veda_sparse_attention_host(_ptr(q), _ptr(k), _ptr(v), q.stride(0), q.stride(1), lat, cfg, Hh, d,
                                              self.k, ctypes.byref(self.scorer), heads_per_chunk, _ptr(out),
                                              _ptr(self._host_ws), self._host_ws.numel(), s),
               "sparse_attention_host")
        return out


def sparse_attention(q, k, v, lat, cfgs, scorer_weights, sparsity=None, k_keep=None):
    """One-shot convenience: the five steps on [Hh, N, d] bf16 CUDA views -> o [Hh, N, d].

    CPU (pinned) inputs go through veda_sparse_attention_host (H2D, the five steps and
    D2H pipelined over head chunks) and the output is returned on the host."""
    Hh, N, d = q.shape
    if not q.is_cuda:  # host tensors: the pipelined end-to-end entry point
        dev = torch.device("cuda")
        scorer_weights = {n: w.to(dev) for n, w in scorer_weights.items()}
        path = SparseAttention(lat, cfgs, Hh, d, scorer_weights, sparsity=sparsity, k=k_keep, device=dev)
        o = path.run_host(q, k, v)
        torch.cuda.current_stream().synchronize()
        return o
    path = SparseAttention(lat, cfgs, Hh, d, scorer_weights, sparsity=sparsity, k=k_keep, device=q.device)
    return path(q, k, v)
