/*
 * TEST INFRASTRUCTURE — CPU numerical oracle (see oracle_numerics.h for the
 * scope statement: the reference has no numerical path, so the numerics are
 * pinned against transformers' Mixtral, tests/test_oracle_golden_hf.py).  Every function cites the paper / reference line it
 * restates.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
 * load this library.
 */
#include "oracle_numerics.h"

#include <immintrin.h>
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* bf16 + synthetic weights (SURVEY.md §8c "Synthetic weights")            */
/* ---------------------------------------------------------------------- */
float orc_bf16_to_f32(uint16_t v) {
    uint32_t u = (uint32_t)v << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

uint16_t orc_f32_to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u); /* round to nearest even */
    return (uint16_t)(u >> 16);
}

static inline float rb(float f) { return orc_bf16_to_f32(orc_f32_to_bf16(f)); }

static inline uint64_t mix64(uint64_t z) { /* splitmix64 finalizer */
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_tensor_id(int layer, int kind, int expert) {
    return ((uint64_t)(layer + 1) << 16) | ((uint64_t)kind << 8) | (uint64_t)expert;
}

void orc_gen_bf16(uint64_t seed, uint64_t tid, int64_t n, float scale, int is_norm,
                  uint16_t* out) {
    const uint64_t key = mix64(seed ^ mix64(tid));
    const float a = (float)(1.7320508075688772 * (double)scale);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t h = mix64(key + (uint64_t)i);
        const float r = 2.0f * ((float)(h >> 40) * 0x1p-24f) - 1.0f; /* exact, [-1, 1) */
        out[i] = orc_f32_to_bf16(is_norm ? 1.0f + r * 0.1f : r * a);
    }
}

/* ---------------------------------------------------------------------- */
/* kernels                                                                  */
/* ---------------------------------------------------------------------- */

/* Every dot product of the oracle has one fixed summation structure: 16
 * lane partials p_j = sum over k = j (mod 16), in k order, each step one
 * fused multiply-add (fp32, single rounding); then s = p_0 + p_1 + ... +
 * p_15 left to right; then the K % 16 tail in order.  dot16 is the scalar
 * statement of it; the blocked AVX-512 paths below evaluate exactly the same
 * operations (one zmm lane per partial), so they are bit-identical to it and
 * to each other for any blocking and thread count. */
static inline float dot16(const float* x, const float* w, int n) {
    float acc[16] = {0};
    int k = 0;
    for (; k + 16 <= n; k += 16)
        for (int j = 0; j < 16; ++j) acc[j] = fmaf(x[k + j], w[k + j], acc[j]);
    float s = 0.0f;
    for (int j = 0; j < 16; ++j) s += acc[j];
    for (; k < n; ++k) s = fmaf(x[k], w[k], s);
    return s;
}

static inline float hsum16(__m512 v) {
    float a[16];
    _mm512_storeu_ps(a, v);
    float s = 0.0f;
    for (int j = 0; j < 16; ++j) s += a[j];
    return s;
}

static inline __m512 ld_bf16x16(const uint16_t* p) {
    const __m256i h = _mm256_loadu_si256((const __m256i*)p);
    return _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(h), 16));
}

/* y[t][m] = dot(x[t], w[m]) for 4 weight rows x 4 tokens per register
 * block (16 zmm accumulators; weights widened from bf16 in registers). */
void orc_linear(const float* x, const uint16_t* w, int T, int K, int M, float* y) {
    const int K16 = K & ~15;
#pragma omp parallel for schedule(static)
    for (int m0 = 0; m0 < M; m0 += 4) {
        const uint16_t* wr[4];
        for (int r = 0; r < 4; ++r) wr[r] = w + (size_t)(m0 + r < M ? m0 + r : M - 1) * K;
        for (int t0 = 0; t0 < T; t0 += 4) {
            const float* xr[4];
            for (int t = 0; t < 4; ++t) xr[t] = x + (size_t)(t0 + t < T ? t0 + t : T - 1) * K;
            __m512 acc[4][4];
            for (int r = 0; r < 4; ++r)
                for (int t = 0; t < 4; ++t) acc[r][t] = _mm512_setzero_ps();
            for (int k = 0; k < K16; k += 16) {
                __m512 wv[4];
                for (int r = 0; r < 4; ++r) wv[r] = ld_bf16x16(wr[r] + k);
                for (int t = 0; t < 4; ++t) {
                    const __m512 xv = _mm512_loadu_ps(xr[t] + k);
                    for (int r = 0; r < 4; ++r) acc[r][t] = _mm512_fmadd_ps(xv, wv[r], acc[r][t]);
                }
            }
            for (int r = 0; r < 4 && m0 + r < M; ++r)
                for (int t = 0; t < 4 && t0 + t < T; ++t) {
                    float s = hsum16(acc[r][t]);
                    for (int k = K16; k < K; ++k) s = fmaf(xr[t][k], orc_bf16_to_f32(wr[r][k]), s);
                    y[(size_t)(t0 + t) * M + m0 + r] = s;
                }
        }
    }
}

/* Reference statement of orc_linear (tests pin the blocked path to it). */
void orc_linear_scalar(const float* x, const uint16_t* w, int T, int K, int M, float* y) {
    float* row = (float*)malloc(sizeof(float) * (size_t)K);
    for (int m = 0; m < M; ++m) {
        for (int k = 0; k < K; ++k) row[k] = orc_bf16_to_f32(w[(size_t)m * K + k]);
        for (int t = 0; t < T; ++t) y[(size_t)t * M + m] = dot16(x + (size_t)t * K, row, K);
    }
    free(row);
}

/* RMSNorm, Mixtral convention: y = x / sqrt(mean(x^2) + eps) * gamma. */
void orc_rmsnorm(const float* x, const uint16_t* gamma, int T, int H, float eps, int round_bf16,
                 float* out) {
    for (int t = 0; t < T; ++t) {
        const float* xr = x + (size_t)t * H;
        float ss = 0.0f;
        for (int i = 0; i < H; ++i) ss += xr[i] * xr[i];
        const float r = 1.0f / sqrtf(ss / (float)H + eps);
        for (int i = 0; i < H; ++i) {
            const float v = xr[i] * r * orc_bf16_to_f32(gamma[i]);
            out[(size_t)t * H + i] = round_bf16 ? rb(v) : v;
        }
    }
}

/* Rotate-half RoPE: pairs (i, i + d/2), inv_freq_i = theta^(-2i/d) in
 * double, angle = pos * inv_freq in double, cos/sin rounded to float. */
void orc_rope(float* x, const int32_t* pos, int T, int n_heads, int d, float theta) {
    const int half = d / 2;
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < half; ++i) {
            const double inv = pow((double)theta, -2.0 * (double)i / (double)d);
            const double ang = (double)pos[t] * inv;
            const float c = (float)cos(ang), s = (float)sin(ang);
            for (int h = 0; h < n_heads; ++h) {
                float* v = x + ((size_t)t * n_heads + h) * d;
                const float a = v[i], b = v[i + half];
                v[i] = a * c - b * s;
                v[i + half] = b * c + a * s;
            }
        }
}

/* GQA decode attention ("CPU attention = the softmax
 * part"; reference cost: opcost.cpp:5-15). */
void orc_attention(const float* q, const uint16_t* k, const uint16_t* v, const int32_t* ctx,
                   int T, int n_q, int n_kv, int d, int ctx_cap, float* out) {
    const int group = n_q / n_kv;
    const float scale = 1.0f / sqrtf((float)d);
    /* one work item per (token, query head): scores s_j = dot16(q, k_j) (the
     * oracle's dot structure; d % 16 == 0 is vectorised, else scalar), fp32
     * softmax with expf, o = sum_j p_j v_j accumulated in key order, / l */
#pragma omp parallel for collapse(2) schedule(static)
    for (int t = 0; t < T; ++t)
        for (int h = 0; h < n_q; ++h) {
            const int kh = h / group;
            const int L = ctx[t];
            const float* qv = q + ((size_t)t * n_q + h) * d;
            float* p = (float*)malloc(sizeof(float) * (size_t)(L > 0 ? L : 1) + sizeof(float) * (size_t)d * 2);
            float* kf = p + (L > 0 ? L : 1);
            float* o = out + ((size_t)t * n_q + h) * d;
            float mx = -INFINITY;
            for (int j = 0; j < L; ++j) {
                const uint16_t* kr = k + (((size_t)t * ctx_cap + j) * n_kv + kh) * d;
                float s;
                if ((d & 15) == 0) {
                    __m512 acc = _mm512_setzero_ps();
                    for (int i = 0; i < d; i += 16)
                        acc = _mm512_fmadd_ps(_mm512_loadu_ps(qv + i), ld_bf16x16(kr + i), acc);
                    s = hsum16(acc);
                } else {
                    for (int i = 0; i < d; ++i) kf[i] = orc_bf16_to_f32(kr[i]);
                    s = dot16(qv, kf, d);
                }
                p[j] = s * scale;
                if (p[j] > mx) mx = p[j];
            }
            float l = 0.0f;
            for (int j = 0; j < L; ++j) {
                p[j] = expf(p[j] - mx);
                l += p[j];
            }
            for (int i = 0; i < d; ++i) o[i] = 0.0f;
            for (int j = 0; j < L; ++j) {
                const uint16_t* vr = v + (((size_t)t * ctx_cap + j) * n_kv + kh) * d;
                int i = 0;
                if ((d & 15) == 0) {
                    const __m512 pj = _mm512_set1_ps(p[j]);
                    for (; i < d; i += 16)
                        _mm512_storeu_ps(o + i, _mm512_fmadd_ps(pj, ld_bf16x16(vr + i), _mm512_loadu_ps(o + i)));
                }
                for (; i < d; ++i) o[i] = fmaf(p[j], orc_bf16_to_f32(vr[i]), o[i]);
            }
            const float inv = L > 0 ? 1.0f / l : 0.0f;
            for (int i = 0; i < d; ++i) o[i] *= inv;
            free(p);
        }
}

/* Router: logits in fp32 with a FIXED reduction tree —
 * lane l of 32 accumulates 8-element chunks c = l, l+32, ... with fmaf in
 * element order, then a xor-butterfly over m = 16,8,4,2,1.  top-k on the
 * logits (softmax is monotone), ties to the lower expert index; weights =
 * softmax over the k selected logits; permutation = stable sort by
 * (expert, token, slot).  The GPU kernel (router.cu) mirrors this exactly. */
void orc_router_logits(const uint16_t* hn, const uint16_t* w, int T, int H, int E, float* logits) {
    const int chunks = H / 8;
    for (int t = 0; t < T; ++t)
        for (int e = 0; e < E; ++e) {
            float lane[32];
            for (int l = 0; l < 32; ++l) {
                float acc = 0.0f;
                for (int c = l; c < chunks; c += 32)
                    for (int j = 0; j < 8; ++j)
                        acc = fmaf(orc_bf16_to_f32(hn[(size_t)t * H + c * 8 + j]),
                                   orc_bf16_to_f32(w[(size_t)e * H + c * 8 + j]), acc);
                lane[l] = acc;
            }
            for (int m = 16; m >= 1; m >>= 1) {
                float nxt[32];
                for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ m];
                memcpy(lane, nxt, sizeof lane);
            }
            logits[(size_t)t * E + e] = lane[0];
        }
}

/* Weights (softmax over the k chosen logits, slot order) and the stable
 * (expert, token, slot) permutation for given top-k choices. */
void orc_route(const float* logits, const int32_t* topk_idx, int T, int E, int K, float* topk_w,
               int32_t* perm, int32_t* offsets) {
    for (int t = 0; t < T; ++t) {
        const float* lg = logits + (size_t)t * E;
        const float top = lg[topk_idx[(size_t)t * K]];
        float sum = 0.0f;
        for (int s = 0; s < K; ++s) {
            const float v = expf(lg[topk_idx[(size_t)t * K + s]] - top);
            topk_w[(size_t)t * K + s] = v;
            sum += v;
        }
        for (int s = 0; s < K; ++s) topk_w[(size_t)t * K + s] /= sum;
    }
    for (int e = 0; e <= E; ++e) offsets[e] = 0;
    for (int i = 0; i < T * K; ++i) offsets[topk_idx[i] + 1]++;
    for (int e = 0; e < E; ++e) offsets[e + 1] += offsets[e];
    int fill[64];
    for (int e = 0; e < E; ++e) fill[e] = offsets[e];
    for (int t = 0; t < T; ++t)
        for (int s = 0; s < K; ++s) perm[fill[topk_idx[(size_t)t * K + s]]++] = t * K + s;
}

void orc_router(const uint16_t* hn, const uint16_t* w, int T, int H, int E, int K,
                float* logits, int32_t* topk_idx, float* topk_w, int32_t* perm,
                int32_t* offsets) {
    orc_router_logits(hn, w, T, H, E, logits);
    for (int t = 0; t < T; ++t) {
        const float* lg = logits + (size_t)t * E;
        int used[64] = {0};
        for (int s = 0; s < K; ++s) {
            int best = -1;
            for (int e = 0; e < E; ++e)
                if (!used[e] && (best < 0 || lg[e] > lg[best])) best = e;
            used[best] = 1;
            topk_idx[(size_t)t * K + s] = best;
        }
    }
    orc_route(logits, topk_idx, T, E, K, topk_w, perm, offsets);
}

/* Expert FFN: W2 (silu(x W1^T) * (x W3^T)). */
void orc_expert(const float* x, const uint16_t* w1, const uint16_t* w3, const uint16_t* w2,
                int T, int H, int F, int round_bf16, float* y) {
    float* g = (float*)malloc(sizeof(float) * (size_t)T * F);
    float* u = (float*)malloc(sizeof(float) * (size_t)T * F);
    orc_linear(x, w1, T, H, F, g);
    orc_linear(x, w3, T, H, F, u);
    for (size_t i = 0; i < (size_t)T * F; ++i) {
        const float a = g[i] / (1.0f + expf(-g[i])) * u[i];
        g[i] = round_bf16 ? rb(a) : a;
    }
    orc_linear(g, w2, T, F, H, y);
    free(g);
    free(u);
}

/* ---------------------------------------------------------------------- */
/* whole model                                                              */
/* ---------------------------------------------------------------------- */
struct orc_model {
    orc_config c;
    int d;
    uint16_t *embed, *lm_head, *final_norm;
    uint16_t **attn_norm, **ffn_norm, **wqkv, **wo, **router;
    uint16_t ***w1, ***w3, ***w2;
    uint16_t **kc, **vc; /* [layer] -> [N][max_ctx][n_kv][d] */
    float* rmargin;      /* [N]: min over layers of the router's k-th minus (k+1)-th logit */
    const int32_t* force_topk; /* [L][N][K] routes to take instead of the own top-k (borrowed) */
    int32_t* own_topk;   /* [L][N][K] the oracle's own top-k of the last step */
    float* own_gap;      /* [L][N] its k-th selected minus best unselected logit */
};

static uint16_t* gen(const orc_model* m, int layer, int kind, int expert, int64_t n, double scale,
                     int is_norm) {
    uint16_t* p = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
    orc_gen_bf16(m->c.seed, orc_tensor_id(layer, kind, expert), n, (float)scale, is_norm, p);
    return p;
}

orc_model* orc_model_create(const orc_config* cfg) {
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    m->c = *cfg;
    const int H = cfg->hidden, F = cfg->ffn, L = cfg->layers, E = cfg->experts;
    m->d = H / cfg->q_heads;
    const int qkv = (cfg->q_heads + 2 * cfg->kv_heads) * m->d;
    const double sH = 1.0 / sqrt((double)H), sF = 1.0 / sqrt((double)F);
    m->embed = gen(m, -1, ORC_T_EMBED, 0, (int64_t)cfg->vocab * H, 1.0, 0);
    m->lm_head = gen(m, -1, ORC_T_LM_HEAD, 0, (int64_t)cfg->vocab * H, cfg->lm_head_scale * sH, 0);
    m->final_norm = gen(m, -1, ORC_T_FINAL_NORM, 0, H, 0, 1);
    m->attn_norm = calloc(L, sizeof(void*));
    m->ffn_norm = calloc(L, sizeof(void*));
    m->wqkv = calloc(L, sizeof(void*));
    m->wo = calloc(L, sizeof(void*));
    m->router = calloc(L, sizeof(void*));
    m->w1 = calloc(L, sizeof(void*));
    m->w3 = calloc(L, sizeof(void*));
    m->w2 = calloc(L, sizeof(void*));
    m->kc = calloc(L, sizeof(void*));
    m->vc = calloc(L, sizeof(void*));
    m->rmargin = calloc(cfg->batch, sizeof(float));
    m->own_topk = calloc((size_t)L * cfg->batch * cfg->top_k, sizeof(int32_t));
    m->own_gap = calloc((size_t)L * cfg->batch, sizeof(float));
    const size_t kv = (size_t)cfg->batch * cfg->max_ctx * cfg->kv_heads * m->d;
    for (int l = 0; l < L; ++l) {
        m->attn_norm[l] = gen(m, l, ORC_T_ATTN_NORM, 0, H, 0, 1);
        m->ffn_norm[l] = gen(m, l, ORC_T_FFN_NORM, 0, H, 0, 1);
        m->wqkv[l] = gen(m, l, ORC_T_WQKV, 0, (int64_t)qkv * H, sH, 0);
        m->wo[l] = gen(m, l, ORC_T_WO, 0, (int64_t)H * H, sH, 0);
        m->router[l] = gen(m, l, ORC_T_ROUTER, 0, (int64_t)E * H, sH, 0);
        m->w1[l] = calloc(E, sizeof(void*));
        m->w3[l] = calloc(E, sizeof(void*));
        m->w2[l] = calloc(E, sizeof(void*));
        for (int e = 0; e < E; ++e) {
            m->w1[l][e] = gen(m, l, ORC_T_W1, e, (int64_t)F * H, sH, 0);
            m->w3[l][e] = gen(m, l, ORC_T_W3, e, (int64_t)F * H, sH, 0);
            m->w2[l][e] = gen(m, l, ORC_T_W2, e, (int64_t)H * F, sF, 0);
        }
        m->kc[l] = calloc(kv, sizeof(uint16_t));
        m->vc[l] = calloc(kv, sizeof(uint16_t));
    }
    return m;
}

void orc_model_free(orc_model* m) {
    if (!m) return;
    for (int l = 0; l < m->c.layers; ++l) {
        free(m->attn_norm[l]); free(m->ffn_norm[l]); free(m->wqkv[l]); free(m->wo[l]);
        free(m->router[l]);
        for (int e = 0; e < m->c.experts; ++e) {
            free(m->w1[l][e]); free(m->w3[l][e]); free(m->w2[l][e]);
        }
        free(m->w1[l]); free(m->w3[l]); free(m->w2[l]); free(m->kc[l]); free(m->vc[l]);
    }
    free(m->attn_norm); free(m->ffn_norm); free(m->wqkv); free(m->wo); free(m->router);
    free(m->w1); free(m->w3); free(m->w2); free(m->kc); free(m->vc);
    free(m->embed); free(m->lm_head); free(m->final_norm); free(m->rmargin);
    free(m->own_topk); free(m->own_gap);
    free(m);
}

void orc_router_margins(const orc_model* m, float* out) {
    memcpy(out, m->rmargin, sizeof(float) * (size_t)m->c.batch);
}

void orc_model_force_routes(orc_model* m, const int32_t* topk) { m->force_topk = topk; }

void orc_model_route_info(const orc_model* m, int32_t* own_topk, float* own_gap) {
    const size_t rows = (size_t)m->c.layers * m->c.batch;
    if (own_topk) memcpy(own_topk, m->own_topk, sizeof(int32_t) * rows * m->c.top_k);
    if (own_gap) memcpy(own_gap, m->own_gap, sizeof(float) * rows);
}

const uint16_t* orc_model_tensor(const orc_model* m, int layer, int kind, int expert) {
    switch (kind) {
        case ORC_T_EMBED: return m->embed;
        case ORC_T_LM_HEAD: return m->lm_head;
        case ORC_T_FINAL_NORM: return m->final_norm;
        case ORC_T_ATTN_NORM: return m->attn_norm[layer];
        case ORC_T_FFN_NORM: return m->ffn_norm[layer];
        case ORC_T_WQKV: return m->wqkv[layer];
        case ORC_T_WO: return m->wo[layer];
        case ORC_T_ROUTER: return m->router[layer];
        case ORC_T_W1: return m->w1[layer][expert];
        case ORC_T_W3: return m->w3[layer][expert];
        case ORC_T_W2: return m->w2[layer][expert];
    }
    return 0;
}

/* Element count of a model tensor (the shapes of orc_model_create). */
static int64_t tensor_elems(const orc_model* m, int kind) {
    const orc_config* c = &m->c;
    const int64_t H = c->hidden, F = c->ffn, qkv = (int64_t)(c->q_heads + 2 * c->kv_heads) * m->d;
    switch (kind) {
        case ORC_T_EMBED: case ORC_T_LM_HEAD: return (int64_t)c->vocab * H;
        case ORC_T_FINAL_NORM: case ORC_T_ATTN_NORM: case ORC_T_FFN_NORM: return H;
        case ORC_T_WQKV: return qkv * H;
        case ORC_T_WO: return H * H;
        case ORC_T_ROUTER: return (int64_t)c->experts * H;
        case ORC_T_W1: case ORC_T_W3: case ORC_T_W2: return F * H;
    }
    return 0;
}

int orc_model_set_tensor(orc_model* m, int layer, int kind, int expert, const uint16_t* data) {
    uint16_t* dst = (uint16_t*)orc_model_tensor(m, layer, kind, expert);
    const int64_t n = tensor_elems(m, kind);
    if (!dst || n <= 0) return -1;
    memcpy(dst, data, sizeof(uint16_t) * (size_t)n);
    return 0;
}

uint16_t* orc_model_kv(orc_model* m, int layer, int which) {
    return which ? m->vc[layer] : m->kc[layer];
}

/* Synthetic prompt-stage KV (BASELINE.md "Config 2"): uniform(-1,1) bf16.
 * Element (seq, pos, head, i) is drawn at index ((seq<<20 | pos) * n_kv*d +
 * head*d + i) of tensor (layer, kind 11/12) — independent of capacity. */
void orc_fill_kv(orc_model* m, uint64_t seed, int upto) {
    const int nkd = m->c.kv_heads * m->d;
    for (int l = 0; l < m->c.layers; ++l)
        for (int which = 0; which < 2; ++which) {
            const uint64_t key = mix64(seed ^ mix64(orc_tensor_id(l, 11 + which, 0)));
            uint16_t* dst = which ? m->vc[l] : m->kc[l];
#pragma omp parallel for collapse(2)
            for (int s = 0; s < m->c.batch; ++s)
                for (int p = 0; p < upto; ++p)
                    for (int i = 0; i < nkd; ++i) {
                        const uint64_t idx = (((uint64_t)s << 20) | (uint64_t)p) * nkd + i;
                        const uint64_t h = mix64(key + idx);
                        const float r = 2.0f * ((float)(h >> 40) * 0x1p-24f) - 1.0f;
                        dst[((size_t)s * m->c.max_ctx + p) * nkd + i] = orc_f32_to_bf16(r);
                    }
        }
}

/* One decoder layer for all N sequences (PreAttn = norm +
 * QKV; attention; PostAttn = O projection + MoE FFN). */
int orc_layer_forward(orc_model* m, int layer, float* x, const int32_t* pos, int mode,
                      int32_t* topk_out) {
    const orc_config* c = &m->c;
    const int N = c->batch, H = c->hidden, F = c->ffn, E = c->experts, K = c->top_k, d = m->d;
    const int nq = c->q_heads, nkv = c->kv_heads, W = (nq + 2 * nkv) * d;
    const int faithful = mode == ORC_FAITHFUL;
    for (int t = 0; t < N; ++t)
        if (pos[t] < 0 || pos[t] >= c->max_ctx) return -1;

    float* xn = malloc(sizeof(float) * (size_t)N * H);
    float* qkv = malloc(sizeof(float) * (size_t)N * W);
    float* q = malloc(sizeof(float) * (size_t)N * nq * d);
    float* kk = malloc(sizeof(float) * (size_t)N * nkv * d);
    float* o = malloc(sizeof(float) * (size_t)N * H);
    float* h = malloc(sizeof(float) * (size_t)N * H);
    int32_t* ctx = malloc(sizeof(int32_t) * N);

    orc_rmsnorm(x, m->attn_norm[layer], N, H, c->rms_eps, faithful, xn);
    orc_linear(xn, m->wqkv[layer], N, H, W, qkv);
    for (int t = 0; t < N; ++t) {
        memcpy(q + (size_t)t * nq * d, qkv + (size_t)t * W, sizeof(float) * nq * d);
        memcpy(kk + (size_t)t * nkv * d, qkv + (size_t)t * W + nq * d, sizeof(float) * nkv * d);
    }
    orc_rope(q, pos, N, nq, d, c->rope_theta);
    orc_rope(kk, pos, N, nkv, d, c->rope_theta);
    for (int t = 0; t < N; ++t) {
        if (faithful)
            for (int i = 0; i < nq * d; ++i) q[(size_t)t * nq * d + i] = rb(q[(size_t)t * nq * d + i]);
        const size_t slot = ((size_t)t * c->max_ctx + pos[t]) * nkv * d;
        for (int i = 0; i < nkv * d; ++i) {
            m->kc[layer][slot + i] = orc_f32_to_bf16(kk[(size_t)t * nkv * d + i]);
            m->vc[layer][slot + i] = orc_f32_to_bf16(qkv[(size_t)t * W + (nq + nkv) * d + i]);
        }
        ctx[t] = pos[t] + 1;
    }
    orc_attention(q, m->kc[layer], m->vc[layer], ctx, N, nq, nkv, d, c->max_ctx, o);
    if (faithful)
        for (size_t i = 0; i < (size_t)N * H; ++i) o[i] = rb(o[i]);
    orc_linear(o, m->wo[layer], N, H, H, h);
    for (size_t i = 0; i < (size_t)N * H; ++i) h[i] += x[i];

    /* PostAttn: norm -> router -> experts -> weighted combine + residual */
    float* hn = xn; /* reuse */
    orc_rmsnorm(h, m->ffn_norm[layer], N, H, c->rms_eps, faithful, hn);
    uint16_t* hb = malloc(sizeof(uint16_t) * (size_t)N * H);
    for (size_t i = 0; i < (size_t)N * H; ++i) hb[i] = orc_f32_to_bf16(hn[i]);
    float* logits = malloc(sizeof(float) * (size_t)N * E);
    int32_t* idx = malloc(sizeof(int32_t) * (size_t)N * K);
    float* wts = malloc(sizeof(float) * (size_t)N * K);
    int32_t* perm = malloc(sizeof(int32_t) * (size_t)N * K);
    int32_t* off = malloc(sizeof(int32_t) * (E + 1));
    orc_router(hb, m->router[layer], N, H, E, K, logits, idx, wts, perm, off);
    memcpy(m->own_topk + (size_t)layer * N * K, idx, sizeof(int32_t) * N * K);
    for (int t = 0; t < N; ++t) { /* routing robustness: gap between selected and next logit */
        const float kth = logits[(size_t)t * E + idx[t * K + K - 1]];
        float next = -INFINITY;
        for (int e = 0; e < E; ++e) {
            int sel = 0;
            for (int s = 0; s < K; ++s) sel |= idx[t * K + s] == e;
            if (!sel && logits[(size_t)t * E + e] > next) next = logits[(size_t)t * E + e];
        }
        const float gap = kth - next;
        m->own_gap[(size_t)layer * N + t] = gap;
        if (layer == 0 || gap < m->rmargin[t]) m->rmargin[t] = gap;
    }
    if (m->force_topk) { /* take the given routes (e.g. the GPU's) on the oracle's own logits */
        memcpy(idx, m->force_topk + (size_t)layer * N * K, sizeof(int32_t) * N * K);
        for (int i = 0; i < N * K; ++i)
            if (idx[i] < 0 || idx[i] >= E) {
                free(xn); free(qkv); free(q); free(kk); free(o); free(h); free(ctx); free(hb);
                free(logits); free(idx); free(wts); free(perm); free(off);
                return -1;
            }
        orc_route(logits, idx, N, E, K, wts, perm, off);
    }
    if (topk_out) memcpy(topk_out, idx, sizeof(int32_t) * N * K);

    float* y = malloc(sizeof(float) * (size_t)N * K * H); /* per (t, s) */
    for (int e = 0; e < E; ++e) {
        const int cnt = off[e + 1] - off[e];
        if (!cnt) continue;
        float* xe = malloc(sizeof(float) * (size_t)cnt * H);
        float* ye = malloc(sizeof(float) * (size_t)cnt * H);
        for (int r = 0; r < cnt; ++r)
            memcpy(xe + (size_t)r * H, hn + (size_t)(perm[off[e] + r] / K) * H, sizeof(float) * H);
        orc_expert(xe, m->w1[layer][e], m->w3[layer][e], m->w2[layer][e], cnt, H, F, faithful, ye);
        for (int r = 0; r < cnt; ++r)
            memcpy(y + (size_t)perm[off[e] + r] * H, ye + (size_t)r * H, sizeof(float) * H);
        free(xe);
        free(ye);
    }
    for (int t = 0; t < N; ++t)
        for (int i = 0; i < H; ++i) {
            float acc = 0.0f;
            for (int s = 0; s < K; ++s) acc += wts[t * K + s] * y[((size_t)t * K + s) * H + i];
            x[(size_t)t * H + i] = h[(size_t)t * H + i] + acc;
        }
    free(xn); free(qkv); free(q); free(kk); free(o); free(h); free(ctx); free(hb);
    free(logits); free(idx); free(wts); free(perm); free(off); free(y);
    return 0;
}

int orc_decode_step(orc_model* m, const int32_t* tokens, const int32_t* pos, int mode,
                    int32_t* next, float* margin, float* x_out) {
    const orc_config* c = &m->c;
    const int N = c->batch, H = c->hidden, V = c->vocab;
    float* x = malloc(sizeof(float) * (size_t)N * H);
    for (int t = 0; t < N; ++t) {
        if (tokens[t] < 0 || tokens[t] >= V) { free(x); return -1; }
        for (int i = 0; i < H; ++i)
            x[(size_t)t * H + i] = orc_bf16_to_f32(m->embed[(size_t)tokens[t] * H + i]);
    }
    for (int l = 0; l < c->layers; ++l)
        if (orc_layer_forward(m, l, x, pos, mode, 0)) { free(x); return -1; }
    if (x_out) memcpy(x_out, x, sizeof(float) * (size_t)N * H);
    float* xf = malloc(sizeof(float) * (size_t)N * H);
    float* lg = malloc(sizeof(float) * (size_t)N * V);
    orc_rmsnorm(x, m->final_norm, N, H, c->rms_eps, mode == ORC_FAITHFUL, xf);
    orc_linear(xf, m->lm_head, N, H, V, lg);
    for (int t = 0; t < N; ++t) {
        const float* r = lg + (size_t)t * V;
        int b = 0;
        for (int v = 1; v < V; ++v)
            if (r[v] > r[b]) b = v;
        float second = -INFINITY;
        for (int v = 0; v < V; ++v)
            if (v != b && r[v] > second) second = r[v];
        next[t] = b;
        if (margin) margin[t] = r[b] - second;
    }
    free(x); free(xf); free(lg);
    return 0;
}

int orc_num_threads(void) { return omp_get_max_threads(); }
