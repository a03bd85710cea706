// Host-side launch interface of the sm_100a kernels (namespace mltk).  The
// C ABI (capi/kernels_capi.cpp) and the runtime call only these.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mltk {

enum { kEpiF32 = 0, kEpiSiluPacked = 1 };

struct GemmArgs {
    // A operand: page table of 128-row weight blocks, [n_mats][G][RB].
    const uint8_t* const* a_table = nullptr;
    int n_mats = 1;  // 2 = fused gate/up
    int G = 1;       // groups (experts)
    int RB = 0;      // 128-row blocks per matrix
    int K = 0;       // reduction length (multiple of 64)
    // B operand: packed activations with row capacity R.
    const uint8_t* b = nullptr;
    int R = 0;
    const int32_t* b_off = nullptr;  // [G+1] padded row offset per group (nullptr: dense)
    const int32_t* b_cnt = nullptr;  // [G] valid rows per group (nullptr: dense)
    int rows_dense = 0;              // rows when b_cnt == nullptr
    int n_cap = 16;                  // max tokens per tile (16..256, multiple of 16)
    int n_chunks = 1;                // token chunks per (group, row block) spread over CTAs:
                                     // virtual tile (rb, g, c) handles tokens c*n_cap, +n_chunks*n_cap, ...
    int k_splits = 1;                // split-K: partial s of the fp32 output goes to
    int64_t split_stride = 0;        // out_f32 + s*split_stride (residual ignored; consumer reduces)
    // optional in-kernel timing: [0] = min over CTAs of the %globaltimer at
    // entry, [1] = ~(max at exit); both pre-set to all ones by the caller
    unsigned long long* timing = nullptr;
    // optional per-CTA phase stamps [gridDim][8] (diagnostic, see mlt.h)
    unsigned long long* trace = nullptr;
    // 1: A row blocks are encoded tiles (runtime/weight_codec.hpp, 12432 B
    // per 64-k tile); decoder warps expand them in shared memory.
    // 3: row-plane encoded tiles; decoder warps expand them into tensor
    // memory, the MMA reads its A operand from TMEM (gemm_tc.cu)
    int codec = 0;
    int dec_groups = 2;  // codec 1: decoder groups of 4 warps, each owning every dec_groups-th stage
    // codec 2 (fragment-order tiles, gemm_codec.cu: decode in registers,
    // mma.sync): 1 when some page-table entry of this GEMM is a raw fallback
    // block (tag bit 0; 16 KiB ring slots instead of 12432 B)
    int codec_raw = 0;
    // codec 4: stored bytes of one encoded tile (runtime/weight_codec.hpp
    // codec4_tile_bytes(capacity), sized per weight kind); 0 -> 11600
    int enc_tile = 0;
    // optional CTA-0 pipeline trace [4][256] (%globaltimer): producer issue,
    // decoder start, decoder done, MMA start per k-block (diagnostic)
    unsigned long long* ktrace = nullptr;
    // epilogue
    int epi = kEpiF32;
    float alpha = 1.0f;
    float* out_f32 = nullptr;  // [row][ldo], row = b_off[g] + n
    int ldo = 0;
    const float* residual = nullptr;  // added in kEpiF32 (same row indexing)
    int ldr = 0;
    uint8_t* out_packed = nullptr;  // kEpiSiluPacked: packed B layout, capacity out_R
    int out_R = 0;
    // stream-K tail (kEpiSiluPacked, k_splits == n_chunks == 1, only when the
    // caller provides the scratch): the G*RB % grid tiles of a partial last
    // wave are split along K into sk_parts parts over the whole grid; each
    // part stores its fp32 g/u accumulators to sk_scratch, waits for the
    // tile's other parts (all CTAs are resident: grid = #SMs, one CTA per
    // SM), then sums every part in part order for its slice of the tile's
    // rows and runs the SiLU epilogue.  sk_full / sk_tail / sk_parts are set
    // by launch_gemm.
    float* sk_scratch = nullptr;  // [grid][n_mats][sk_rows][128] fp32
    unsigned long long* sk_count = nullptr;  // [grid] 64-bit monotonic arrival counters, zeroed once
    int sk_rows = 0;              // row capacity per (tile, part): max rows of one group
    int sk_full = 0, sk_tail = 0, sk_parts = 0;
    // filled by launch_gemm
    int stages = 0, acc_stages = 0, tmem_cols = 0;
    int kps = 1;  // k-blocks per ring stage
    // codec 3 rings (stages = encoded-A smem slots): TMEM A slots, token-tile slots, A slot bytes
    int t3_slots = 0, b3_slots = 0, a3_slot_bytes = 0;
};

// Dispatches codec = 2 to launch_gemm_codec (gemm_codec.cu).
cudaError_t launch_gemm(GemmArgs a, int num_sms, cudaStream_t stream);
cudaError_t launch_gemm_codec(GemmArgs a, int num_sms, cudaStream_t stream);

// Programmatic dependent launch for every kernel of this build (see
// common.cuh); off by default; the runtime turns it on for all-GPU schedules.
void set_pdl(bool on);
int gemm_smem_bytes(int n_mats, int n_cap, int stages, int kps = 1);

// x_out[t][:] = float(table[tokens[t]][:])
cudaError_t launch_embed(const int32_t* tokens, const uint16_t* table, int T, int H, float* x_out,
                         cudaStream_t s);

// RMSNorm(x) * gamma -> bf16, written in packed B layout (capacity R rows).
cudaError_t launch_rmsnorm_pack(const float* x, const uint16_t* gamma, int T, int H, float eps,
                                uint8_t* out_packed, int R, cudaStream_t s);

// Row-major bf16 [T, K] -> packed B layout (capacity R).
cudaError_t launch_pack_rows(const uint16_t* src, int ld, int T, int K, uint8_t* dst, int R,
                             cudaStream_t s);

// RoPE (rotate-half) on the q and k parts of qkv fp32 [T, (nq+2nkv)d] using
// cos/sin table [max_pos][d/2] (float2), output bf16 [T, (nq+2nkv)d] rows
// (q | k | v): the D1 offload layout.  qkv may hold `parts` split-K partials
// at qkv + p*part_stride; they are summed first.
// With kv (A_g = 1) the roped k and the v rows are also stored into the
// swizzled paged pool at position pos[t] of sequence kv->seq[t] (fused
// kv_append; d = 128, 16-token pages).
struct KvAppend {
    uint16_t* k_pool = nullptr;
    uint16_t* v_pool = nullptr;
    const int32_t* block_table = nullptr;  // [seq][max_pages]
    int max_pages = 0;
    const int32_t* seq = nullptr;          // [T]
};
cudaError_t launch_rope_qkv(const float* qkv, int parts, int64_t part_stride, const int32_t* pos,
                            const float2* rope, int T, int nq, int nkv, int d, uint16_t* out,
                            cudaStream_t s, const KvAppend* kv = nullptr);

// Router (SURVEY.md §2c router_topk_permute, first half): optional fused
// RMSNorm (x fp32 + gamma) or direct bf16 input; logits with the fixed lane
// tree of oracle orc_router; top-k + softmax over the selected logits.
// With `parts` > 0 the input is split-K partials of the O projection:
// h = residual + sum_p x[p*part_stride] is formed first and written to h_out.
cudaError_t launch_router(const float* x, const uint16_t* gamma, float eps,
                          const uint16_t* hn_in, const uint16_t* w_router, int T, int H, int E,
                          int K, uint16_t* hn_out, float* logits, int32_t* topk_idx,
                          float* topk_w, cudaStream_t s, int parts = 0, int64_t part_stride = 0,
                          const float* residual = nullptr, float* h_out = nullptr);

// Stable (expert, token, slot) permutation with per-expert 16-row padding
// and gather of hn rows into the packed expert operand X (capacity R rows).
// counts[E], offsets[E+1] (padded), perm[R] (padded row -> t*K+s, -1 pad),
// inv[T*K] (slot -> padded row).
cudaError_t launch_moe_permute(const int32_t* topk_idx, const uint16_t* hn, int T, int H, int E,
                               int K, int32_t* counts, int32_t* offsets, int32_t* perm,
                               int32_t* inv, uint8_t* x_packed, int R, cudaStream_t s);

// x_out[t] = h[t] + sum_s w[t,s] * y[inv[t*K+s]]  (fp32, slot order).
// With gamma: also RMSNorm(x_out) * gamma -> packed bf16 xn (capacity R),
// the operand of the next projection (fused next-layer / final norm).
cudaError_t launch_moe_combine(const float* h, const float* y, int ldy, const int32_t* inv,
                               const float* topk_w, int T, int H, int K, float* x_out,
                               cudaStream_t s, const uint16_t* gamma = nullptr, float eps = 0.f,
                               uint8_t* xn = nullptr, int R = 0, int n_parts = 1, int64_t part_stride = 0);

// out[i] = sum_p parts[p*stride + i] (+ add[i]); n % 4 == 0.  Fixed order.
cudaError_t launch_sum_parts(const float* parts, int n_parts, int64_t stride, const float* add,
                             float* out, int64_t n, cudaStream_t s);

// Greedy ids: argmax (ties -> lower index) of fp32 logits [T, V]; margin =
// top1 - top2 (optional).
cudaError_t launch_argmax(const float* logits, int T, int V, int32_t* ids, float* margin,
                          cudaStream_t s);

// GQA decode attention over a paged KV cache (SURVEY.md §2c
// gqa_decode_paged).  KV pages hold `page` tokens x n_kv heads x d (bf16),
// K and V in separate pools; block_table[seq][max_pages]; ctx[t] tokens
// of sequence seq[t].  q bf16 rows with leading dimension ldq (the rope
// output [T, (nq+2nkv)d] works directly); output written in packed B layout
// (capacity R) for the O projection and/or fp32 row-major.
// Split-KV scratch: splits = S (0: auto, the count in 1..max_splits that best
// fills whole waves), scratch >= T * nq * max_splits * 130 floats, counters
// >= T * nkv ints zeroed once (each launch leaves them zero).
struct GqaSplit {
    int splits = 0;
    int max_splits = 8;
    float* scratch = nullptr;
    int* counters = nullptr;
};
// Stream-K decode (attention.cu gqa_decode_flat_kernel): ctas = gqa_flat_ctas(#SMs)
// resident CTAs split the flattened (token, kv head, page) space evenly;
// scratch >= ctas * 4 warps * 2 slots * G * 130 floats, counters >= T * nkv
// ints zeroed once (every launch leaves them zero).  Same output.
struct GqaFlat {
    int ctas = 0;
    float* scratch = nullptr;
    int* counters = nullptr;
};
int gqa_flat_ctas(int num_sms);
cudaError_t launch_gqa_decode_flat(const uint16_t* q, int ldq, const uint16_t* k_pool, const uint16_t* v_pool,
                                   const int32_t* block_table, int max_pages, const int32_t* seq, const int32_t* ctx,
                                   int T, int nq, int nkv, int d, int page, uint8_t* out_packed, int R,
                                   float* out_rowmajor, const GqaFlat& fl, cudaStream_t s);
cudaError_t launch_gqa_decode_paged(const uint16_t* q, int ldq, const uint16_t* k_pool,
                                    const uint16_t* v_pool, const int32_t* block_table,
                                    int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                                    int nq, int nkv, int d, int page, uint8_t* out_packed, int R,
                                    float* out_rowmajor, cudaStream_t s, const GqaSplit* split = nullptr);

// Append this step's k/v (bf16 rows from the rope output [T, (nq+2nkv)d])
// into the paged cache at position ctx[t]-1 of sequence seq[t].
cudaError_t launch_kv_append(const uint16_t* qkv_bf16, int nq, int nkv, int d,
                             const int32_t* seq, const int32_t* pos, int T,
                             const int32_t* block_table, int max_pages, int page,
                             uint16_t* k_pool, uint16_t* v_pool, cudaStream_t s);

// ---- prefill (attention_prefill.cu) --------------------------------------
// Causal GQA over a chunk of whole prompt sequences.  qkv: roped bf16 rows
// [T][W]; tiles[i] = {first row of the sequence, its length, first query
// position (multiple of 16)}; one CTA per (tile, kv head).  Output: packed
// bf16 operand (capacity R) of the O projection.
cudaError_t launch_prefill_attention(const uint16_t* qkv, int W, const int4* tiles, int n_tiles, int nq,
                                     int nkv, int d, uint8_t* out_packed, int R, cudaStream_t s);
// K/V rows -> per-sequence [n_kv][len][d] staging (sequence s at row
// seq_row0[s] * n_kv * d) for one strided D2H copy per sequence.
cudaError_t launch_kv_stage(const uint16_t* qkv, int W, int nq, int nkv, int d, const int32_t* tok_seq,
                            const int32_t* tok_pos, const int32_t* seq_row0, const int32_t* seq_len, int T,
                            uint16_t* stage_k, uint16_t* stage_v, cudaStream_t s);
// dst[i] = x[idx[i]] (fp32 rows of width H).
cudaError_t launch_gather_rows(const float* x, const int32_t* idx, int n, int H, float* dst, cudaStream_t s);

}  // namespace mltk
