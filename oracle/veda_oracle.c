/*
 * veda_oracle.c -- fp64 CPU oracle for the Veda tile-sparse attention hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2605_30325_b200/csrc); it is
 * written from the paper (arXiv 2605.30325, /root/reference/PAPER.md) alone.
 *
 * Every routine is a plain loop nest in the paper's order and notation, in fp64.
 * There is no blocking, fusion or reordering beyond what the cited passage states.
 * bf16 inputs are taken as raw 16-bit patterns and widened exactly to fp64.
 *
 * Readings where the paper is silent are DESIGN.md "Readings" R1..R17 (they follow
 * SURVEY.md §8(c) c2); each routine names the readings it relies on.
 *
 * Parity pins (tests/test_oracle_pins.py) tie every routine to something other than
 * itself: worked examples, closed forms, invariants and library special cases.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* exact widening of a bf16 bit pattern */
static double bf16_to_f64(uint16_t b)
{
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* ------------------------------------------------------------------------- *
 * c1.1  Padded grid.  PAPER.md:143-145 (§3.1: "N tokens are grouped into N_T
 * tiles of size B"), PAPER.md:288-294 (Eq. 8: p_t p_h p_w = B, one config per
 * head).  Reading R4/R5: each axis is zero-padded up to a multiple of the
 * largest tile extent used on that axis by any head, so N_T is the same for
 * every head.  PAPER.md:471 fixes 61x45x80 -> 245,760 tokens = 64x48x80.
 * out[0..4] = T', H', W', B, N_T.   Returns 0 on success.
 * ------------------------------------------------------------------------- */
int vo_grid(int T, int H, int W, const int32_t *cfg, int Hh, int64_t *out)
{
    if (T < 1 || H < 1 || W < 1 || Hh < 1) return 1;
    int64_t B = (int64_t)cfg[0] * cfg[1] * cfg[2];
    int Pt = 1, Ph = 1, Pw = 1;
    for (int h = 0; h < Hh; ++h) {
        const int32_t *c = cfg + 3 * h;
        if (c[0] < 1 || c[1] < 1 || c[2] < 1) return 2;
        if ((int64_t)c[0] * c[1] * c[2] != B) return 3;
        /* lcm of the extents (they are powers of two in practice, so lcm = max) */
        int a;
        a = Pt; while (a % c[0]) a += Pt; Pt = a;
        a = Ph; while (a % c[1]) a += Ph; Ph = a;
        a = Pw; while (a % c[2]) a += Pw; Pw = a;
    }
    int64_t Tp = ((T + Pt - 1) / Pt) * (int64_t)Pt;
    int64_t Hp = ((H + Ph - 1) / Ph) * (int64_t)Ph;
    int64_t Wp = ((W + Pw - 1) / Pw) * (int64_t)Pw;
    out[0] = Tp; out[1] = Hp; out[2] = Wp; out[3] = B;
    out[4] = Tp * Hp * Wp / B;
    return 0;
}

/* ------------------------------------------------------------------------- *
 * c1.2  Tiling.  PAPER.md:133 (N = THW, raster flatten, reading R1),
 * PAPER.md:143-145 (tiled tensors Q~,K~,V~ in R^{N_T x B x d}),
 * PAPER.md:290 (pi_{l,h} = (p_t,p_h,p_w) per head), Alg. 2 PAPER.md:685-686.
 * Tile order: raster over boxes (R2); slot order inside a box: raster
 * (dt,dh,dw) (R3, consistent with PAPER.md:610 "temporal neighbours satisfy
 * |phi_tile(u)-phi_tile(v)| <= p_h p_w").  Padded slots hold +0 (R4).
 *   x      : [Hh][N][d] bf16 bits, element (h,n,c) at x[h*hs + n*ts + c]
 *   xt     : [Hh][N_T][B][d]
 *   cnt    : [Hh][N_T] number of real tokens in the tile (may be NULL)
 *   mask   : [Hh][N_T][ceil(B/32)] bit b set iff slot b holds a real token (may be NULL)
 * ------------------------------------------------------------------------- */
int vo_tile_permute(const uint16_t *x, int64_t hs, int64_t ts, int T, int H, int W,
                    const int32_t *cfg, int Hh, int d, uint16_t *xt, int32_t *cnt,
                    uint32_t *mask)
{
    int64_t g[5];
    int rc = vo_grid(T, H, W, cfg, Hh, g);
    if (rc) return rc;
    const int64_t Hp = g[1], Wp = g[2], B = g[3], NT = g[4];
    const int64_t MW = (B + 31) / 32;
    for (int h = 0; h < Hh; ++h) {
        const int pt = cfg[3 * h], ph = cfg[3 * h + 1], pw = cfg[3 * h + 2];
        const int64_t nbh = Hp / ph, nbw = Wp / pw;
        for (int64_t i = 0; i < NT; ++i) {
            const int64_t it = i / (nbh * nbw), ih = (i / nbw) % nbh, iw = i % nbw;
            int32_t c_valid = 0;
            if (mask) memset(mask + (h * NT + i) * MW, 0, MW * sizeof(uint32_t));
            for (int64_t j = 0; j < B; ++j) {
                const int64_t dt = j / (ph * pw), dh = (j / pw) % ph, dw = j % pw;
                const int64_t t = it * pt + dt, hh = ih * ph + dh, w = iw * pw + dw;
                uint16_t *dst = xt + ((h * NT + i) * B + j) * d;
                if (t < T && hh < H && w < W) {
                    const int64_t n = (t * H + hh) * W + w;
                    const uint16_t *src = x + h * hs + n * ts;
                    for (int c = 0; c < d; ++c) dst[c] = src[c];
                    ++c_valid;
                    if (mask) mask[(h * NT + i) * MW + j / 32] |= 1u << (j % 32);
                } else {
                    for (int c = 0; c < d; ++c) dst[c] = 0;
                }
            }
            if (cnt) cnt[h * NT + i] = c_valid;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- *
 * c1.8  UnTiling.  Alg. 1 PAPER.md:660 ("after mapping tokens back to the
 * original order").  Inverse of vo_tile_permute on real slots;
 * padded slots are dropped (R4).
 * ------------------------------------------------------------------------- */
int vo_tile_unpermute(const uint16_t *xt, int T, int H, int W, const int32_t *cfg, int Hh,
                      int d, uint16_t *x, int64_t hs, int64_t ts)
{
    int64_t g[5];
    int rc = vo_grid(T, H, W, cfg, Hh, g);
    if (rc) return rc;
    const int64_t Hp = g[1], Wp = g[2], B = g[3], NT = g[4];
    for (int h = 0; h < Hh; ++h) {
        const int pt = cfg[3 * h], ph = cfg[3 * h + 1], pw = cfg[3 * h + 2];
        const int64_t nbh = Hp / ph, nbw = Wp / pw;
        for (int64_t i = 0; i < NT; ++i) {
            const int64_t it = i / (nbh * nbw), ih = (i / nbw) % nbh, iw = i % nbw;
            for (int64_t j = 0; j < B; ++j) {
                const int64_t dt = j / (ph * pw), dh = (j / pw) % ph, dw = j % pw;
                const int64_t t = it * pt + dt, hh = ih * ph + dh, w = iw * pw + dw;
                if (t < T && hh < H && w < W) {
                    const int64_t n = (t * H + hh) * W + w;
                    const uint16_t *src = xt + ((h * NT + i) * B + j) * d;
                    uint16_t *dst = x + h * hs + n * ts;
                    for (int c = 0; c < d; ++c) dst[c] = src[c];
                }
            }
        }
    }
    return 0;
}

static int slot_valid(const uint32_t *mask_tile, int64_t b)
{
    return (mask_tile[b / 32] >> (b % 32)) & 1u;
}

/* ------------------------------------------------------------------------- *
 * c1.3  TripPool, Eq. 5: PAPER.md:261-265 ("concatenating {Avg, Max, Min}
 * triplet statistics"), Alg. 2 PAPER.md:689-690.  Per tile and channel, over
 * the tile's real tokens (R7): z = Avg (+) Max (+) Min, width 3d, in that order
 * (R6).  A tile with no real token gets z = 0 (R5).
 *   xt [Hh][N_T][B][d] bf16 bits, mask as produced by vo_tile_permute
 *   z  [Hh][N_T][3d] fp64
 * ------------------------------------------------------------------------- */
void vo_trippool(const uint16_t *xt, const uint32_t *mask, int Hh, int64_t NT, int B,
                 int d, double *z)
{
    const int64_t MW = (B + 31) / 32;
    for (int64_t ti = 0; ti < (int64_t)Hh * NT; ++ti) {
        const uint32_t *mk = mask + ti * MW;
        double *zz = z + ti * 3 * d;
        for (int c = 0; c < d; ++c) {
            double sum = 0.0, mx = -INFINITY, mn = INFINITY;
            int64_t n = 0;
            for (int64_t b = 0; b < B; ++b) {
                if (!slot_valid(mk, b)) continue;
                const double v = bf16_to_f64(xt[(ti * B + b) * d + c]);
                sum += v;
                if (v > mx) mx = v;
                if (v < mn) mn = v;
                ++n;
            }
            if (n == 0) { zz[c] = 0.0; zz[d + c] = 0.0; zz[2 * d + c] = 0.0; continue; }
            zz[c] = sum / (double)n;      /* Avg */
            zz[d + c] = mx;               /* Max */
            zz[2 * d + c] = mn;           /* Min */
        }
    }
}

/* GELU(x) = x * Phi(x) = 0.5 x (1 + erf(x / sqrt 2))   (reading R8) */
static double gelu(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }

/* ------------------------------------------------------------------------- *
 * c1.4  Head-specific projection phi, Eq. 6: PAPER.md:266-270 ("head-specific
 * MLP projections phi_q and phi_k ... distinct projection weights are learned
 * for each head"), Alg. 2 PAPER.md:693-694.  Reading R8: two-layer MLP
 *     e = GELU(z W1 + b1) W2 + b2,
 * W1 [Hh][din][dh], b1 [Hh][dh], W2 [Hh][dh][dl], b2 [Hh][dl] (fp32 weights,
 * widened exactly to fp64).  z [Hh][N_T][din], e [Hh][N_T][dl].
 * ------------------------------------------------------------------------- */
void vo_mlp(const double *z, int Hh, int64_t NT, int din, int dh, int dl, const float *W1,
            const float *b1, const float *W2, const float *b2, double *e)
{
    double *u = (double *)malloc(sizeof(double) * (size_t)dh);
    for (int h = 0; h < Hh; ++h) {
        const float *w1 = W1 + (int64_t)h * din * dh, *w2 = W2 + (int64_t)h * dh * dl;
        const float *bb1 = b1 + (int64_t)h * dh, *bb2 = b2 + (int64_t)h * dl;
        for (int64_t i = 0; i < NT; ++i) {
            const double *zi = z + ((int64_t)h * NT + i) * din;
            double *ei = e + ((int64_t)h * NT + i) * dl;
            for (int m = 0; m < dh; ++m) {
                double a = 0.0;
                for (int c = 0; c < din; ++c) a += zi[c] * (double)w1[(int64_t)c * dh + m];
                u[m] = gelu(a + (double)bb1[m]);
            }
            for (int n = 0; n < dl; ++n) {
                double a = 0.0;
                for (int m = 0; m < dh; ++m) a += u[m] * (double)w2[(int64_t)m * dl + n];
                ei[n] = a + (double)bb2[n];
            }
        }
    }
    free(u);
}

/* ------------------------------------------------------------------------- *
 * c1.5  Tile-pair scores, Eq. 6: PAPER.md:267-269
 *     S_pred_ij = phi_q(z_q,i) . phi_k(z_k,j)^T / sqrt(d')
 * Alg. 2 PAPER.md:695.  Reading R5: a key tile with no real token scores -inf.
 *   eq, ek [Hh][N_T][dl];  cnt_k [Hh][N_T];  s [Hh][N_T][N_T]
 * ------------------------------------------------------------------------- */
void vo_scores(const double *eq, const double *ek, const int32_t *cnt_k, int Hh, int64_t NT,
               int dl, double *s)
{
    const double rs = sqrt((double)dl);
    for (int h = 0; h < Hh; ++h)
        for (int64_t i = 0; i < NT; ++i)
            for (int64_t j = 0; j < NT; ++j) {
                double *out = s + ((int64_t)h * NT + i) * NT + j;
                if (cnt_k[(int64_t)h * NT + j] == 0) { *out = -INFINITY; continue; }
                const double *a = eq + ((int64_t)h * NT + i) * dl;
                const double *b = ek + ((int64_t)h * NT + j) * dl;
                double acc = 0.0;
                for (int c = 0; c < dl; ++c) acc += a[c] * b[c];
                *out = acc / rs;
            }
}

/* ------------------------------------------------------------------------- *
 * c1.6  Per-query-tile Top-k.  PAPER.md:146-149 (exactly k kept key tiles per
 * query tile), PAPER.md:280 ("retain the k highest-scoring key tiles for each
 * query tile"), Alg. 2 PAPER.md:697.  Reading R10: exactly k, ties go to the
 * lower key-tile index; R11: emitted ascending.  Literally: order the key
 * tiles by (S descending, j ascending), take the first k, sort them by j.
 *   s [rows][ncols] (fp64; callers pass fp32-rounded values, reading R15)
 *   idx [rows][k]
 * ------------------------------------------------------------------------- */
static const double *g_row; /* comparator context (single-threaded use) */
static int cmp_desc_then_index(const void *pa, const void *pb)
{
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    const double sa = g_row[a], sb = g_row[b];
    if (sa > sb) return -1;
    if (sa < sb) return 1;
    return (a > b) - (a < b);
}
static int cmp_int(const void *pa, const void *pb)
{
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    return (a > b) - (a < b);
}
int vo_topk(const double *s, int64_t rows, int64_t ncols, int k, int32_t *idx)
{
    if (k < 1 || k > ncols) return 4;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)ncols);
    for (int64_t r = 0; r < rows; ++r) {
        g_row = s + r * ncols;
        for (int64_t j = 0; j < ncols; ++j) order[j] = (int32_t)j;
        qsort(order, (size_t)ncols, sizeof(int32_t), cmp_desc_then_index);
        int32_t *out = idx + r * k;
        memcpy(out, order, sizeof(int32_t) * (size_t)k);
        qsort(out, (size_t)k, sizeof(int32_t), cmp_int);
    }
    free(order);
    return 0;
}

/* ------------------------------------------------------------------------- *
 * c1.7  Tile-sparse attention, Eq. 2: PAPER.md:150-157
 *     K^_i = Concat_{j: M_ij=1} K~_j ,  V^_i = Concat_{j: M_ij=1} V~_j
 *     O_i  = Softmax(Q~_i K^_i^T / sqrt(d)) V^_i
 * with the additive-mask reading of PAPER.md:140,145 for padded slots (R4):
 * a padded key slot is left out of K^_i (equivalently -inf), a padded query
 * slot yields O = 0.  Softmax is max-subtracted (R14); scale is 1/sqrt(d)
 * unless the caller passes another positive value.
 *   qt,kt,vt [Hh][N_T][B][d] bf16 bits;  idx [Hh][N_T][k];  mask as above
 *   units: optional list of unit ids u = h*N_T + i to compute (NULL = all);
 *          outputs of units not listed are left untouched
 *   o   [Hh][N_T][B][d] fp64;  lse [Hh][N_T][B] fp64 natural log (may be NULL)
 * ------------------------------------------------------------------------- */
typedef struct {
    const uint16_t *qt, *kt, *vt;
    const int32_t *idx;
    const uint32_t *mask;
    int64_t NT;
    int B, d, k;
    double scale;
    const int64_t *units;
    int64_t n_units;
    double *o, *lse;
    int64_t next; /* shared work counter */
    pthread_mutex_t mu;
} attn_job;

static void attn_unit(attn_job *J, int64_t u, double *logit, int64_t *key_row)
{
    const int B = J->B, d = J->d, k = J->k;
    const int64_t NT = J->NT, MW = (B + 31) / 32;
    const int64_t h = u / NT;
    /* K^_i, V^_i: rows of the kept tiles, in list order, real slots only */
    int64_t nk = 0;
    for (int t = 0; t < k; ++t) {
        const int64_t j = J->idx[u * k + t];
        const uint32_t *mk = J->mask + (h * NT + j) * MW;
        for (int b = 0; b < B; ++b)
            if (slot_valid(mk, b)) key_row[nk++] = (h * NT + j) * B + b;
    }
    const uint32_t *mq = J->mask + u * MW;
    for (int a = 0; a < B; ++a) {
        double *o = J->o + (u * B + a) * d;
        if (!slot_valid(mq, a) || nk == 0) {
            for (int c = 0; c < d; ++c) o[c] = 0.0;
            if (J->lse) J->lse[u * B + a] = -INFINITY;
            continue;
        }
        const uint16_t *q = J->qt + (u * B + a) * d;
        double mx = -INFINITY;
        for (int64_t r = 0; r < nk; ++r) {
            const uint16_t *kk = J->kt + key_row[r] * d;
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += bf16_to_f64(q[c]) * bf16_to_f64(kk[c]);
            logit[r] = acc * J->scale;
            if (logit[r] > mx) mx = logit[r];
        }
        double z = 0.0;
        for (int64_t r = 0; r < nk; ++r) { logit[r] = exp(logit[r] - mx); z += logit[r]; }
        for (int c = 0; c < d; ++c) o[c] = 0.0;
        for (int64_t r = 0; r < nk; ++r) {
            const double p = logit[r] / z;
            const uint16_t *vv = J->vt + key_row[r] * d;
            for (int c = 0; c < d; ++c) o[c] += p * bf16_to_f64(vv[c]);
        }
        if (J->lse) J->lse[u * B + a] = mx + log(z);
    }
}

static void *attn_worker(void *arg)
{
    attn_job *J = (attn_job *)arg;
    const int64_t cap = (int64_t)J->k * J->B;
    double *logit = (double *)malloc(sizeof(double) * (size_t)cap);
    int64_t *key_row = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= J->n_units) break;
        attn_unit(J, J->units ? J->units[w] : w, logit, key_row);
    }
    free(logit);
    free(key_row);
    return NULL;
}

int vo_sparse_attn(const uint16_t *qt, const uint16_t *kt, const uint16_t *vt,
                   const int32_t *idx, const uint32_t *mask, int Hh, int64_t NT, int B, int d,
                   int k, double scale, const int64_t *units, int64_t n_units, double *o,
                   double *lse, int nthreads)
{
    if (k < 1 || k > NT) return 4;
    attn_job J;
    J.qt = qt; J.kt = kt; J.vt = vt; J.idx = idx; J.mask = mask;
    J.NT = NT; J.B = B; J.d = d; J.k = k;
    J.scale = scale > 0 ? scale : 1.0 / sqrt((double)d);
    J.units = units;
    J.n_units = units ? n_units : (int64_t)Hh * NT;
    J.o = o; J.lse = lse; J.next = 0;
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, attn_worker, &J);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    return 0;
}

/* ------------------------------------------------------------------------- *
 * NEXT-2a  Target tile scores, Eq. 4: PAPER.md:253-258 (section 4.1)
 *     A* = Softmax(Q K^T / sqrt(d)),   S_tgt_ij = max_{(u,v) in Tile(i,j)} A*_uv
 * (Alg. 3 "MaxPool(A*, kernel=B, stride=B)").  Reading R4: the softmax runs
 * over the real keys of the whole sequence; padded query slots are dropped from the
 * max; a key tile without real tokens scores -inf (as in S_pred, R5); a query tile
 * without real tokens gets a row of 0 (its outputs are discarded anyway).
 *   qt, kt [Hh][N_T][B][d] bf16 bits; mask [Hh][N_T][MW]; s [Hh][N_T][N_T] fp64
 *   units: optional list of query tiles u = h*N_T + i to compute (NULL = all)
 * ------------------------------------------------------------------------- */
typedef struct {
    const uint16_t *qt, *kt;
    const uint32_t *mask;
    int64_t NT;
    int B, d;
    double scale;
    const int64_t *units;
    int64_t n_units;
    double *s;
    int64_t next;
    pthread_mutex_t mu;
} tgt_job;

static void tgt_unit(tgt_job *J, int64_t u, double *logit)
{
    const int B = J->B, d = J->d;
    const int64_t NT = J->NT, MW = (B + 31) / 32, h = u / NT;
    double *row = J->s + u * NT;
    for (int64_t j = 0; j < NT; ++j) {
        int any = 0;
        for (int b = 0; b < B; ++b) any |= slot_valid(J->mask + (h * NT + j) * MW, b);
        row[j] = any ? 0.0 : -INFINITY;
    }
    const uint32_t *mq = J->mask + u * MW;
    for (int a = 0; a < B; ++a) {
        if (!slot_valid(mq, a)) continue;
        const uint16_t *q = J->qt + (u * B + a) * d;
        /* full softmax over every real key of head h */
        double mx = -INFINITY;
        for (int64_t j = 0; j < NT; ++j)
            for (int b = 0; b < B; ++b) {
                double *l = logit + j * B + b;
                if (!slot_valid(J->mask + (h * NT + j) * MW, b)) { *l = -INFINITY; continue; }
                const uint16_t *kk = J->kt + ((h * NT + j) * B + b) * d;
                double acc = 0.0;
                for (int c = 0; c < d; ++c) acc += bf16_to_f64(q[c]) * bf16_to_f64(kk[c]);
                *l = acc * J->scale;
                if (*l > mx) mx = *l;
            }
        double z = 0.0;
        for (int64_t r = 0; r < NT * B; ++r)
            if (logit[r] != -INFINITY) z += exp(logit[r] - mx);
        /* max-pool of A*_uv over each key tile */
        for (int64_t j = 0; j < NT; ++j)
            for (int b = 0; b < B; ++b) {
                const double l = logit[j * B + b];
                if (l == -INFINITY) continue;
                const double p = exp(l - mx) / z;
                if (p > row[j]) row[j] = p;
            }
    }
}

static void *tgt_worker(void *arg)
{
    tgt_job *J = (tgt_job *)arg;
    double *logit = (double *)malloc(sizeof(double) * (size_t)(J->NT * J->B));
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= J->n_units) break;
        tgt_unit(J, J->units ? J->units[w] : w, logit);
    }
    free(logit);
    return NULL;
}

void vo_target_scores(const uint16_t *qt, const uint16_t *kt, const uint32_t *mask, int Hh, int64_t NT, int B,
                      int d, double scale, const int64_t *units, int64_t n_units, double *s, int nthreads)
{
    tgt_job J;
    J.qt = qt; J.kt = kt; J.mask = mask; J.NT = NT; J.B = B; J.d = d;
    J.scale = scale > 0 ? scale : 1.0 / sqrt((double)d);
    J.units = units; J.n_units = units ? n_units : (int64_t)Hh * NT; J.s = s; J.next = 0;
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, tgt_worker, &J);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
}

/* ------------------------------------------------------------------------- *
 * NEXT-2b  Tile recall, Eq. 3: PAPER.md:225-233 (section 3.2)
 *     Recall@k = (1 / N_T) sum_i |S_i^sp intersect S_i^fu| / k
 * with S^sp the predicted kept set and S^fu the oracle (full-attention) set of query
 * tile i.  Reading R4: the mean runs over query tiles that hold at least one real token
 * (cnt > 0).  Returns the recall; idx lists [rows][k] (any order).
 * ------------------------------------------------------------------------- */
double vo_recall(const int32_t *idx_sp, const int32_t *idx_fu, const int32_t *cnt, int64_t rows, int k)
{
    double acc = 0.0;
    int64_t n = 0;
    for (int64_t r = 0; r < rows; ++r) {
        if (cnt && cnt[r] == 0) continue;
        int inter = 0;
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b)
                if (idx_sp[r * k + a] == idx_fu[r * k + b]) { ++inter; break; }
        acc += (double)inter / (double)k;
        ++n;
    }
    return n ? acc / (double)n : 0.0;
}
