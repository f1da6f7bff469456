// common.cuh -- shared host/device plumbing of libveda (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <functional>

#include "../../include/veda.h"

namespace veda {

// thread-local detail string for veda_last_error()
veda_status fail(veda_status st, const char *fmt, ...);
// count one kernel launch (veda_launch_count)
void count_launch(uint64_t n = 1);
// CUDA error after a launch -> VEDA_ERR_CUDA with the runtime's message
veda_status check_launch(const char *what);
// number of SMs of the current device (cached per device)
int num_sms();
// 2-D bf16 tensor map over a [rows][cols] row-major matrix, SWIZZLE_128B, box {64, box_rows}
veda_status make_tmap_bf16(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols,
                           uint32_t box_rows);

// 5-D bf16 tensor map over a token tensor x[h][n][c] (element strides head_stride,
// token_stride; n = (t*H + h')*W + w) whose box is ONE tile of shape (pt, ph, pw) x 64
// channels: the box lands in smem as pt*ph*pw rows of 128 B in slot order (reading R3),
// SWIZZLE_128B, out-of-grid slots zero-filled (reading R4) -- the same image as a 2-D box
// of the tiled tensor.  Dimension order follows the strides (head-major: d,W,H,T,Hh;
// token-major: d,Hh,W,H,T); *tok_major reports which.
// box_c channels per box (64 with SWIZZLE_128B for the MMA operands; d without swizzle for
// plain row-wise reads).
veda_status make_tmap_tile_tokens(CUtensorMap *map, const void *base, int64_t head_stride, int64_t token_stride,
                                  int Hh, int T, int H, int W, int d, int pt, int ph, int pw, int *tok_major,
                                  int box_c = 64, bool swizzle = true);

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int kMaxHeads = 1024;

// per-head tile configuration packed for kernel parameters
struct HeadCfgs {
    uint8_t pt[kMaxHeads], ph[kMaxHeads], pw[kMaxHeads];
};

// padded grid of a call (readings R4/R5): per-axis lcm of the heads' tile extents
struct Shape {
    int Tp, Hp, Wp, B, NT;
};
veda_status check_arch();
veda_status shape_of(veda_latent lat, const veda_tile_cfg *cfg, int Hh, Shape *sh, HeadCfgs *hc);
size_t align256(size_t v);

// launchers (defined in the per-kernel .cu files)
veda_status launch_tile_permute(const uint16_t *x, int64_t hs, int64_t ts, const HeadCfgs &cf, int Hh,
                                int Tp, int Hp, int Wp, int T, int H, int W, int B, int NT, int d,
                                uint16_t *xt, int32_t *cnt, uint32_t *mask, float *z, cudaStream_t s);
veda_status launch_tile_unpermute(const uint16_t *xt, const HeadCfgs &cf, int Hh, int Tp, int Hp,
                                  int Wp, int T, int H, int W, int B, int NT, int d, uint16_t *x,
                                  int64_t hs, int64_t ts, cudaStream_t s);
veda_status launch_trippool(const uint16_t *xt, const uint32_t *mask, int Hh, int NT, int B, int d,
                            float *z, cudaStream_t s);
veda_status launch_project(const float *z, int Hh, int NT, int din, int dh, int dl, const float *w1,
                           const float *b1, const float *w2, const float *b2, double *hidden,
                           double *e, cudaStream_t s);
veda_status launch_pair_scores(const double *eq, const double *ek, const int32_t *cnt, int Hh, int NT,
                               int dl, float *scores, cudaStream_t s);
veda_status launch_topk(const float *scores, int Hh, int NT, int k, int32_t *idx, cudaStream_t s);
veda_status launch_sparse_attn(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                               const int32_t *idx, const uint32_t *mask, int Hh, int NT, int B, int d,
                               int kk, float scale, uint16_t *o, float *lse, cudaStream_t s);
// attention straight from / to the token layout (no tiled copies)
veda_status launch_sparse_attn_tok(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t hs, int64_t ts,
                                   const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp, int T, int H, int W, int B,
                                   int NT, int d, const int32_t *idx, const uint32_t *mask, int kk, float scale,
                                   uint16_t *o, int64_t o_hs, int64_t o_ts, float *lse, int u_begin, int u_end,
                                   cudaStream_t s);  // units [u_begin, u_end) of the flattened (head, query tile) space
veda_status launch_tile_pool_tokens(const uint16_t *x, int64_t hs, int64_t ts, const HeadCfgs &cf, int Hh, int Tp,
                                    int Hp, int Wp, int T, int H, int W, int B, int NT, int d, float *z,
                                    int32_t *cnt, uint32_t *mask, cudaStream_t s);
// Q and K pooled by one launch (same strides, same grid): z, z2 for x, x2; cnt / mask from x
veda_status launch_tile_pool_tokens2(const uint16_t *x, const uint16_t *x2, int64_t hs, int64_t ts, const HeadCfgs &cf,
                                     int Hh, int Tp, int Hp, int Wp, int T, int H, int W, int B, int NT, int d,
                                     float *z, float *z2, int32_t *cnt, uint32_t *mask, cudaStream_t s);
// scorer GEMMs on the INT8 tensor cores (ozaki.cu); w_q / w_k = {w1, b1, w2, b2}
size_t ozaki_workspace(int Hh, int NT, int din, int dh, int dl);
veda_status launch_ozaki_score(const float *zq, const float *zk, const int32_t *cnt, int Hh, int NT, int din, int dh,
                               int dl, const float *const w_q[4], const float *const w_k[4], const void *prepared,
                               double *hidden, double *eq, double *ek, float *scores, void *scratch, cudaStream_t s);
veda_status launch_ozaki_phi(const float *zq, const float *zk, int Hh, int NT, int din, int dh, int dl,
                             const float *const w_q[4], const float *const w_k[4], const void *prepared,
                             double *hidden, double *eq, double *ek, void *scratch, cudaStream_t s);
size_t ozaki_prepared_bytes(int Hh, int din, int dh, int dl);
veda_status launch_ozaki_prepare(const float *const w_q[4], const float *const w_k[4], int Hh, int din, int dh, int dl,
                                 void *prepared, cudaStream_t s);
veda_status launch_ozaki_pair_scores(const double *eq, const double *ek, const int32_t *cnt, int Hh, int NT, int din,
                                     int dh, int dl, float *scores, void *scratch, cudaStream_t s);
veda_status launch_ozaki_split_e(const double *eq, const double *ek, int Hh, int NT, int din, int dh, int dl,
                                 void *scratch, cudaStream_t s);
veda_status launch_ozaki_score_gemm(const int32_t *cnt, int Hh, int h0, int hn, int NT, int din, int dh, int dl,
                                    float *scores, const void *scratch, cudaStream_t s);
veda_status launch_target_scores(const uint16_t *q, const uint16_t *k, const uint32_t *mask, const float *lse,
                                 int Hh, int NT, int B, int d, float scale, float *out, cudaStream_t s);
veda_status launch_permute_scalar(const float *x, int64_t hs, const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp,
                                  int T, int H, int W, int B, int NT, float pad, float *xt, cudaStream_t s);
veda_status launch_unpermute_scalar(const float *xt, const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp, int T,
                                    int H, int W, int B, int NT, float *x, int64_t hs, cudaStream_t s);
veda_status launch_sq_err(const uint16_t *a, const uint16_t *b, int64_t hs, int64_t n, int Hh, double *err,
                          cudaStream_t s);
veda_status launch_recall(const int32_t *sp, const int32_t *fu, const int32_t *cnt, int64_t rows, int NT, int k,
                          double *recall, cudaStream_t s);

// input validation (validate.cu): kernels that OR VEDA_FLAG_* bits into a device word, and
// debug mode (veda_set_debug / VEDA_DEBUG): run `enqueue(flags)`, synchronise, map flags to
// VEDA_ERR_INDEX / VEDA_ERR_NONFINITE
veda_status launch_validate_index(const int32_t *idx, int64_t rows, int n_tiles, int k, uint32_t *flags,
                                  cudaStream_t s);
veda_status launch_validate_finite(const uint16_t *x, int64_t hs, int64_t ts, int Hh, int64_t n, int d,
                                   uint32_t *flags, cudaStream_t s);
veda_status launch_validate_scores(const float *scores, int64_t n, uint32_t *flags, cudaStream_t s);
veda_status launch_validate_finite_f32(const float *x, int64_t n, uint32_t *flags, cudaStream_t s);
bool debug_mode();
void set_debug_mode(bool on);
veda_status debug_validate(cudaStream_t s, const std::function<veda_status(uint32_t *)> &enqueue);

}  // namespace veda
