"""CPU-only checks of the C ABI: the library builds and loads, exports every symbol
include/veda.h declares, and its host-side logic agrees with the oracle.  No compute
call reaches a GPU here; calls that would need one must fail loudly (VEDA_ERR_CUDA /
VEDA_ERR_ARCH), never silently succeed."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_30325_b200 import build, veda

    build.build()
    return veda.load()


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "veda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(veda_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_2605_30325_b200 import veda

    names = _declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(veda.EXPORTS)


def test_shape_helper_matches_oracle(lib, oracle):
    from paper_2605_30325_b200 import veda

    cases = [((61, 45, 80), [(4, 4, 8)], 24), ((21, 30, 52), [(4, 4, 8)], 12), ((21, 45, 80), [(4, 4, 8)], 40),
             ((4, 8, 8), [(4, 4, 4)], 1), ((9, 10, 13), [(4, 4, 8), (8, 4, 4), (4, 8, 4), (8, 8, 2)], 4),
             ((3, 5, 6), [(4, 4, 4)], 1)]
    for lat, cfgs, Hh in cases:
        sh = veda.tiled_shape(lat, cfgs, Hh)
        full = cfgs * Hh if len(cfgs) == 1 else cfgs
        assert (sh.tp, sh.hp, sh.wp, sh.B, sh.n_tiles) == oracle.grid(lat, full, Hh)
        assert sh.n_pad == sh.tp * sh.hp * sh.wp
    assert veda.tiled_shape((61, 45, 80), [(4, 4, 8)], 24).n_pad == 245760


def test_k_for_sparsity_matches_oracle(lib, oracle):
    from paper_2605_30325_b200 import veda

    for nt in (4, 336, 448, 720, 960, 1920):
        for s in (0.0, 0.5, 0.8, 0.9, 0.95, 0.98, 0.999):
            assert veda.k_for_sparsity(nt, s) == oracle.k_for_sparsity(nt, s)


def test_config_errors(lib):
    from paper_2605_30325_b200 import veda

    with pytest.raises(veda.VedaError, match="CONFIG"):
        veda.tiled_shape((4, 4, 4), [(4, 4, 2), (4, 4, 4)], 2)   # B differs across heads
    with pytest.raises(veda.VedaError, match="CONFIG"):
        veda.tiled_shape((4, 4, 4), [(2, 2, 2)], 1)              # B = 8 unsupported
    with pytest.raises(veda.VedaError, match="CONFIG"):
        veda.tiled_shape((4, 4, 12), [(4, 4, 6)], 1)             # not powers of two (B = 96)
    with pytest.raises(veda.VedaError, match="SHAPE"):
        veda.tiled_shape((0, 4, 4), [(4, 4, 8)], 1)


def test_workspace_query(lib):
    from paper_2605_30325_b200 import veda

    sc = veda.Scorer(384, 768, 128, *([None] * 8))
    n = ctypes.c_size_t(0)
    assert lib.veda_tile_score_workspace(24, 1920, 128, ctypes.byref(sc), ctypes.byref(n)) == 0
    rows = 24 * 1920
    assert n.value >= rows * (2 * 384 * 4 + 768 * 8 + 2 * 128 * 8)
    bad = veda.Scorer(100, 768, 128, *([None] * 8))
    assert lib.veda_tile_score_workspace(24, 1920, 128, ctypes.byref(bad), ctypes.byref(n)) == 2  # SHAPE


def test_argument_errors_without_gpu(lib):
    """Validation happens before any device call; with valid arguments and no GPU the
    call fails loudly (no CPU fallback)."""
    from paper_2605_30325_b200 import veda

    st = lib.veda_select_topk(None, 1, 4, 2, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_NULL"
    fake = ctypes.c_void_p(16)
    st = lib.veda_select_topk(fake, 1, 4, 5, fake, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_K_RANGE"
    st = lib.veda_sparse_attn_fwd(fake, fake, fake, fake, fake, 1, 4, 128, 128, 0, 0.0, fake, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_K_RANGE"
    st = lib.veda_tile_permute(ctypes.c_void_p(17), 0, 128, veda.Latent(4, 4, 8), veda._cfg_array([(4, 4, 8)], 1),
                               1, 128, fake, None, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_ALIGN"
    import torch

    if not torch.cuda.is_available():
        st = lib.veda_select_topk(fake, 1, 4, 2, fake, None)
        assert veda.VEDA_STATUS[st] in ("VEDA_ERR_CUDA", "VEDA_ERR_ARCH")
        assert lib.veda_check_device() != 0
        assert lib.veda_last_error()


def test_binding_refuses_cpu_tensors(lib):
    import torch

    from paper_2605_30325_b200 import veda

    x = torch.zeros((1, 256, 64), dtype=torch.bfloat16)
    with pytest.raises(veda.VedaError, match="no CPU fallback"):
        veda.tile_permute(x, (4, 8, 8), [(4, 4, 4)])


def test_status_strings(lib):
    from paper_2605_30325_b200 import veda

    for i, n in enumerate(veda.VEDA_STATUS):
        assert lib.veda_status_str(i).decode() == n


def test_token_path_and_host_entry_errors(lib):
    """Argument validation of the token-layout entry points and the host pipeline: NULL
    pointers, misaligned strides, k out of range, unsupported layouts and workspace sizing
    (all checked before any device work)."""
    from paper_2605_30325_b200 import veda

    fake = ctypes.c_void_p(256)
    lat = veda.Latent(4, 8, 8)
    cfg = veda._cfg_array([(4, 4, 4)], 1)
    st = lib.veda_tile_pool(None, 16384, 64, lat, cfg, 1, 64, fake, None, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_NULL"
    st = lib.veda_tile_pool(fake, 16384, 63, lat, cfg, 1, 64, fake, None, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_ALIGN"
    st = lib.veda_tile_pool(fake, 16384, 64, lat, cfg, 1, 96, fake, None, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_SHAPE"
    st = lib.veda_sparse_attn_fwd_tokens(fake, fake, fake, 16384, 64, lat, cfg, 1, 64, None, fake, 1, 0.0, fake,
                                         16384, 64, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_NULL"
    st = lib.veda_sparse_attn_fwd_tokens(fake, fake, fake, 16384, 64, lat, cfg, 1, 64, fake, fake, 1, 0.0,
                                         ctypes.c_void_p(258), 16384, 64, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_ALIGN"
    # host pipeline: workspace query validates k and the scorer; layouts must be dense
    w = veda.Scorer(192, 384, 64, *([fake] * 8))
    nb = ctypes.c_size_t(0)
    st = lib.veda_sparse_attention_host_workspace(lat, cfg, 1, 64, 9, ctypes.byref(w), 0, ctypes.byref(nb))
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_K_RANGE"
    st = lib.veda_sparse_attention_host_workspace(lat, cfg, 1, 64, 2, ctypes.byref(w), 0, ctypes.byref(nb))
    assert st == 0 and nb.value > 0
    st = lib.veda_sparse_attention_host(None, fake, fake, 16384, 64, lat, cfg, 1, 64, 2, ctypes.byref(w), 0, fake,
                                        fake, nb.value, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_NULL"


def test_empty_inputs_rejected_before_device_work(lib):
    """Empty problems (no heads, no tiles, an empty latent axis) are argument errors
    (VEDA_ERR_SHAPE), reported identically with or without a GPU: every entry point
    validates shapes before its first device call."""
    from paper_2605_30325_b200 import veda

    fake = ctypes.c_void_p(16)
    lat, cfg = veda.Latent(4, 4, 8), veda._cfg_array([(4, 4, 8)], 1)
    shape = lambda st: veda.VEDA_STATUS[st]  # noqa: E731
    assert shape(lib.veda_select_topk(fake, 0, 4, 2, fake, None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_select_topk(fake, 1, 0, 1, fake, None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_sparse_attn_fwd(fake, fake, fake, fake, fake, 0, 4, 128, 128, 2, 0.1, fake, None,
                                          None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_tile_permute(fake, 0, 128, lat, cfg, 0, 128, fake, None, None, None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_tile_permute(fake, 0, 128, veda.Latent(0, 4, 8), cfg, 1, 128, fake, None, None,
                                       None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_tile_unpermute(fake, lat, cfg, 0, 128, fake, 0, 128, None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_tile_pool(fake, 16384, 128, lat, cfg, 0, 128, fake, fake, fake, None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_tile_pool(fake, 16384, 128, veda.Latent(4, 0, 8), cfg, 1, 128, fake, fake, fake,
                                    None)) == "VEDA_ERR_SHAPE"
    assert shape(lib.veda_tile_pool_heads(fake, 16384, 128, lat, cfg, 1, 128, 0, 2, fake, fake, fake,
                                          None)) == "VEDA_ERR_SHAPE"  # head range beyond Hh
    assert shape(lib.veda_tile_pool_heads(fake, 16384, 128, lat, cfg, 1, 128, 1, 0, fake, fake, fake,
                                          None)) == "VEDA_ERR_SHAPE"  # begin > end


def test_validation_calls_check_arguments_without_a_gpu(lib):
    """veda_validate_index / veda_validate_finite reject bad arguments before any device call;
    veda_set_debug toggles and reports the previous mode."""
    from paper_2605_30325_b200 import veda

    st = lib.veda_validate_index(None, 4, 8, 2, None, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_NULL"
    dummy = ctypes.c_void_p(16)
    st = lib.veda_validate_index(dummy, 4, 8, 9, dummy, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_K_RANGE"
    st = lib.veda_validate_finite(dummy, 64, 8, 1, 8, 7, dummy, None)
    assert veda.VEDA_STATUS[st] == "VEDA_ERR_SHAPE"
    prev = lib.veda_set_debug(1)
    assert lib.veda_set_debug(prev) == 1
