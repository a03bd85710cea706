/*
 * TEST INFRASTRUCTURE — CPU numerical oracle for the MoE decode hot path.
 *
 * NUMERICS PINNED EXTERNALLY, NOT BY THE REFERENCE: the reference artifact
 * (/root/reference/proj, "lightplan") contains no numerical forward pass, no
 * kernels and no golden tensors (proj/README.md:25), and no
 * third-party arithmetic dependency is vendored.  The oracle is instead pinned
 * against Hugging Face transformers' MixtralForCausalLM on its own synthetic
 * weights (tests/golden/mixtral_hf_tiny.npz from tools/make_golden_mixtral.py,
 * tests/test_oracle_golden_hf.py) and against numpy restatements per block
 * (tests/test_oracle_pins.py).  This file restates the decode step from the
 * paper (PAPER.md:143-167 MoE semantics, :385-392 task split) plus public
 * Mixtral conventions (RMSNorm eps 1e-5, rotate-half RoPE theta 1e6, fp32
 * router softmax over the top-k logits, SiLU-gated experts).  It is only
 * ever used as the checker (tests/, __graft_entry__.smoke, bench.py's
 * cpu_baseline / --impl reference legs), never by the product.
 *
 * Two activation modes:
 *   ORC_FP32     fp32 activations everywhere (the "fp32 CPU reference" of
 *                the 2e-2 layer-output tolerance).
 *   ORC_FAITHFUL activations rounded to bf16 at exactly the kernel
 *                boundaries where the GPU stores bf16, so
 *                greedy ids can be compared for 32 steps.
 * The router logit reduction tree is specified exactly (orc_router) and is
 * mirrored bit-for-bit by the GPU router kernel.
 */
#ifndef ORACLE_NUMERICS_H_
#define ORACLE_NUMERICS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FP32 = 0, ORC_FAITHFUL = 1 };

/* Synthetic-weight tensor kinds (tensor id = ((layer+1) << 16) | (kind << 8) | expert). */
enum {
    ORC_T_EMBED = 0, ORC_T_LM_HEAD = 1, ORC_T_FINAL_NORM = 2, ORC_T_ATTN_NORM = 3,
    ORC_T_FFN_NORM = 4, ORC_T_WQKV = 5, ORC_T_WO = 6, ORC_T_ROUTER = 7, ORC_T_W1 = 8,
    ORC_T_W3 = 9, ORC_T_W2 = 10
};

typedef struct orc_config {
    int32_t layers, hidden, ffn, q_heads, kv_heads, experts, top_k, vocab;
    int32_t batch;   /* N sequences */
    int32_t max_ctx; /* KV capacity per sequence */
    float rms_eps, rope_theta, lm_head_scale;
    uint64_t seed;
} orc_config;

uint64_t orc_tensor_id(int layer, int kind, int expert);
/* n bf16 values of tensor `tid`: uniform(-a, a) with a = sqrt(3)*scale
 * (norm gammas: 1 + uniform(-0.1, 0.1)).  Element i depends only on
 * (seed, tid, i). */
void orc_gen_bf16(uint64_t seed, uint64_t tid, int64_t n, float scale, int is_norm,
                  uint16_t* out);
float orc_bf16_to_f32(uint16_t v);
uint16_t orc_f32_to_bf16(float v);

/* Router: logits of T bf16 rows against E bf16 rows (H % 256 == 0) with the
 * fixed lane/butterfly tree, top-k (ties -> lower expert index), softmax over
 * the k selected logits, and the stable (expert, token, slot) permutation.
 * perm[pos] = t*K + s; offsets[E+1]. */
void orc_router(const uint16_t* hn, const uint16_t* w, int T, int H, int E, int K,
                float* logits, int32_t* topk_idx, float* topk_w, int32_t* perm,
                int32_t* offsets);

/* The two halves of orc_router: logits (fixed tree) and, for given top-k
 * choices, the softmax weights + stable permutation. */
void orc_router_logits(const uint16_t* hn, const uint16_t* w, int T, int H, int E, float* logits);
void orc_route(const float* logits, const int32_t* topk_idx, int T, int E, int K, float* topk_w,
               int32_t* perm, int32_t* offsets);

void orc_rmsnorm(const float* x, const uint16_t* gamma, int T, int H, float eps, int round_bf16,
                 float* out);

/* GQA decode attention of T queries over per-sequence KV (bf16), lengths
 * ctx[t].  q [T, n_q*d] fp32; k,v [T][ctx_cap][n_kv][d] bf16; out [T, n_q*d]. */
void orc_attention(const float* q, const uint16_t* k, const uint16_t* v, const int32_t* ctx,
                   int T, int n_q, int n_kv, int d, int ctx_cap, float* out);

/* Dense y = x W^T, x fp32 [T,K], W bf16 [M,K] -> fp32 [T,M].  Each output
 * is one dot product in the oracle's fixed structure (16 lane partials of
 * fused multiply-adds in k order, then summed left to right, then the tail);
 * orc_linear (blocked AVX-512, OpenMP) and orc_linear_scalar (the plain
 * statement) are bit-identical. */
void orc_linear(const float* x, const uint16_t* w, int T, int K, int M, float* y);
void orc_linear_scalar(const float* x, const uint16_t* w, int T, int K, int M, float* y);

/* One expert FFN over T rows: W2 (silu(x W1^T) * (x W3^T)); faithful rounds
 * the intermediate to bf16. */
void orc_expert(const float* x, const uint16_t* w1, const uint16_t* w3, const uint16_t* w2,
                int T, int H, int F, int round_bf16, float* y);

/* Rotary embedding in place on T rows of n_heads*d at positions pos[t]. */
void orc_rope(float* x, const int32_t* pos, int T, int n_heads, int d, float theta);

/* ---- whole model ----------------------------------------------------- */
typedef struct orc_model orc_model;
orc_model* orc_model_create(const orc_config* cfg);
void orc_model_free(orc_model* m);
/* Pointer to a generated weight tensor (bf16, row-major). */
const uint16_t* orc_model_tensor(const orc_model* m, int layer, int kind, int expert);
/* Decode one token for every sequence: tokens[N] at positions pos[N]
 * (KV appended at pos).  Writes greedy ids, the top1-top2 logit margin per
 * sequence, and (optional) the final residual [N,H].  Layers [0, n_layers). */
int orc_decode_step(orc_model* m, const int32_t* tokens, const int32_t* pos, int mode,
                    int32_t* next, float* margin, float* x_out);
/* Per-layer entry for layer-output tolerance tests: x [N,H] fp32 in/out. */
int orc_layer_forward(orc_model* m, int layer, float* x, const int32_t* pos, int mode,
                      int32_t* topk_idx);
/* Fill the KV cache of every layer/sequence for positions [0, upto) with
 * uniform(-1,1) bf16 from `seed` (synthetic prompt-stage KV). */
void orc_fill_kv(orc_model* m, uint64_t seed, int upto);
/* After a decode step / layer forward: per sequence, the smallest gap over
 * layers between the k-th selected router logit and the best unselected one
 * (a routing near-tie indicator). */
void orc_router_margins(const orc_model* m, float* out);
uint16_t* orc_model_kv(orc_model* m, int layer, int which); /* which: 0=K 1=V */
/* Replace a generated tensor with caller weights (same shape, bf16 bits):
 * parity of caller-weight runs (mlt_runtime_create_with_weights). */
int orc_model_set_tensor(orc_model* m, int layer, int kind, int expert, const uint16_t* data);
/* Forced routing (parity probe): with topk != NULL ([L][N][K], borrowed until
 * reset with NULL) every layer takes these experts instead of its own top-k,
 * weighted by the softmax of the ORACLE's logits at those experts.  Lets the
 * residual be compared against a GPU run on the identical route even where a
 * router near-tie flipped; the oracle's own choice is still recorded. */
void orc_model_force_routes(orc_model* m, const int32_t* topk);
/* The last step's own (unforced) top-k [L][N][K] and its gap [L][N]. */
void orc_model_route_info(const orc_model* m, int32_t* own_topk, float* own_gap);
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
