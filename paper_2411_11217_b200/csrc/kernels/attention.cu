// GQA decode attention over a paged KV cache (north_star item 4; SURVEY.md
// §2c gqa_decode_paged), used when the policy places attention on the GPU
// (A_g = 1).  Memory-bound: attention intensity is 2*n_q/(n_kv*dt_kv) FLOP/B
// (4 for 8x7B), so the kernel's job is to stream K/V pages at HBM rate with
// as few instructions per byte as possible.
//
// Layout (common.cuh kv_page_off): a KV page holds kKvPage = 16 tokens of ONE
// kv head, [16][128] bf16 with the 16-byte chunks of token r XOR-swizzled by
// r & 7 (K and V in separate pools), so a (page, head) slice is one
// contiguous 4 KiB run that a single cp.async.bulk moves into shared memory
// and every ldmatrix phase on it is bank-conflict-free.
// Page id = block_table[seq][pos / 16]; pool offset = (id*n_kv + h)*16*128.
//
// One CTA per (query token, kv head).  Its kWarps warps split the pages
// (warp w takes pages w, w+kWarps, ...: flash-decoding inside the CTA); each
// warp owns a kStagesW-deep ring of pages that its elected lane fills with
// 1-D bulk copies (mbarrier tx counts), so the page gather is staged through
// shared memory ahead of the math.  The math runs on the tensor cores
// (mma.sync m16n8k16 bf16 -> fp32) in the transposed orientation, which
// wastes nothing on the token axis and at most half on the head axis:
//   S^T[16 tok][8 heads] = K_page[16][128] . Q^T       (8 MMAs, K by ldmatrix,
//                                                      Q^T fragments in regs,
//                                                      heads >= G are zero)
//   O^T[128][8 heads]   += V_page^T[128][16] . P^T     (V^T by ldmatrix.trans;
//                                                      P^T from the S^T
//                                                      accumulators by
//                                                      movmatrix.trans)
// P is split into bf16 hi + lo parts (two MMAs per tile), so the PV product
// keeps ~16 mantissa bits — fp32-class accuracy at 16 extra MMAs per page.
// Each thread's accumulator columns are heads 2*(lane%4)+{0,1} in both S^T
// and O^T, so the online-softmax rescale is thread-local; the row max needs
// 3 xor-shuffles per page, the row sum is reduced once at the end.  ~100
// instructions per 8 KiB page and warp (vs ~1500 for CUDA-core FMAs).  The
// warps' (m, l, O) are merged through shared memory at the end.
//
// Split-KV (flash-decoding across CTAs): with few (token, kv head) pairs the
// grid is a fraction of a wave (mu = 64: 512 CTAs = 1.73 waves of 2 CTAs x
// 148 SMs), so a token's pages are split S ways over blockIdx.z.  Each split
// CTA stores its unnormalised partial (O, m, l) per head to a scratch, and
// the last split to arrive (a per-(token, head) counter it resets to 0)
// merges all S partials in split order — deterministic for any arrival
// order — and writes the output.
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kPage = kKvPage;
constexpr int kD = 128;
constexpr int kWarps = 4;
constexpr int kStagesW = 3;
constexpr int kPageElems = kPage * kD;
constexpr int kPageBytes = kPageElems * 2;  // 4 KiB (one of K or V)
constexpr int kCombStride = kD + 4;         // per (warp, head): acc[128], m, l, pad
constexpr int kMinSplitPages = 16;          // split-KV auto: fewest pages (256 tokens) per split
constexpr int kMaxFlatTokens = 4096;        // stream-K decode: page-prefix array in smem

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(d) : "r"(a));
    return d;
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(uint16_t lo, uint16_t hi) {
    return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}

// byte offset of 16-byte chunk c of token row r inside a staged page
__device__ __forceinline__ uint32_t pg_off(int r, int c) {
    return static_cast<uint32_t>(r * 256 + ((c ^ (r & 7)) << 4));
}

// One staged (K, V) page of 16 tokens for the warp's G heads: S^T = K Q^T on
// the tensor cores, online softmax (exp2, thread-local rescale), O^T += V^T P^T
// with P split into bf16 hi + lo.  m / l / acc are the warp's running state
// (heads 2tg + {0,1} per thread; l is this thread's tokens only).
__device__ __forceinline__ void page_step(uint32_t sk, uint32_t sv, int ntok, const uint32_t (&qb)[8][2], float sl2,
                                          int lane, float (&m)[2], float (&l)[2], float (&acc)[8][4]) {
    const int g = lane >> 2;
    const int mi = lane >> 3, rr = lane & 7;
    const int k_row = rr + (mi & 1) * 8, k_chunk = mi >> 1;   // K (A, non-trans): [tok][d] blocks
    const int v_row = rr + (mi >> 1) * 8, v_chunk = mi & 1;   // V (A = V^T, trans)
    // ---- S^T = K Q^T: 16 tokens x 8 heads ----
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(sk + pg_off(k_row, 2 * kk + k_chunk), a0, a1, a2, a3);
        mma16816(s, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
    }
    // s[0], s[1]: token g, heads 2tg, 2tg+1; s[2], s[3]: token g+8
    s[0] = g < ntok ? s[0] * sl2 : -INFINITY;
    s[1] = g < ntok ? s[1] * sl2 : -INFINITY;
    s[2] = g + 8 < ntok ? s[2] * sl2 : -INFINITY;
    s[3] = g + 8 < ntok ? s[3] * sl2 : -INFINITY;
    float mx0 = fmaxf(s[0], s[2]), mx1 = fmaxf(s[1], s[3]);
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);  // finite: >= 1 valid token
    const float c0 = exp2f(m[0] - mn0), c1 = exp2f(m[1] - mn1);
    m[0] = mn0;
    m[1] = mn1;
    const float p00 = exp2f(s[0] - mn0), p01 = exp2f(s[1] - mn1);
    const float p10 = exp2f(s[2] - mn0), p11 = exp2f(s[3] - mn1);
    l[0] = l[0] * c0 + p00 + p10;  // this thread's tokens only; lanes reduced at the end
    l[1] = l[1] * c1 + p01 + p11;
    // P^T fragments (k = token, n = head) by transposing the two 8x8 halves
    const uint16_t h00 = f32_to_bf16_bits(p00), h01 = f32_to_bf16_bits(p01);
    const uint16_t h10 = f32_to_bf16_bits(p10), h11 = f32_to_bf16_bits(p11);
    const uint32_t ph0 = movm_t(pack2(h00, h01)), ph1 = movm_t(pack2(h10, h11));
    const uint32_t pl0 = movm_t(pack2(f32_to_bf16_bits(p00 - bf16_bits_to_f32(h00)),
                                      f32_to_bf16_bits(p01 - bf16_bits_to_f32(h01))));
    const uint32_t pl1 = movm_t(pack2(f32_to_bf16_bits(p10 - bf16_bits_to_f32(h10)),
                                      f32_to_bf16_bits(p11 - bf16_bits_to_f32(h11))));
    // ---- O^T += V^T P^T: 8 d-tiles of 16 ----
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        acc[mt][0] *= c0;
        acc[mt][1] *= c1;
        acc[mt][2] *= c0;
        acc[mt][3] *= c1;
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(sv + pg_off(v_row, 2 * mt + v_chunk), a0, a1, a2, a3);
        mma16816(acc[mt], a0, a1, a2, a3, ph0, ph1);
        mma16816(acc[mt], a0, a1, a2, a3, pl0, pl1);
    }
}

template <int G>
__global__ void __launch_bounds__(kWarps * 32) gqa_decode_kernel(
    const uint16_t* __restrict__ q, int ldq, const uint16_t* __restrict__ kp, const uint16_t* __restrict__ vp,
    const int32_t* __restrict__ bt, int max_pages, const int32_t* __restrict__ seq, const int32_t* __restrict__ ctx,
    int nkv, uint8_t* out_p, int R, float* out_f, int S, float* __restrict__ part, int* __restrict__ cnt) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    static_assert(G >= 1 && G <= 8, "heads per kv head must fit the MMA n = 8");
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[kWarps][kStagesW];
    __shared__ int last_split;
    const int t = blockIdx.x, h = blockIdx.y, sp = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int L = ctx[t];
    const int s_id = seq[t];
    const int n_all = (L + kPage - 1) / kPage;
    // this split's pages [p0, p1) of the token's n_all
    const int p0 = static_cast<int>(static_cast<int64_t>(sp) * n_all / S);
    const int n_pages = static_cast<int>(static_cast<int64_t>(sp + 1) * n_all / S);
    // per-warp ring: [warp][stage][K page | V page]
    uint8_t* ring = sm + static_cast<size_t>(warp) * kStagesW * 2 * kPageBytes;
    const uint32_t ring_s = smem_u32(ring);
    // after its loop, each warp's ring holds its partial state [8 heads][kCombStride]
    auto comb = [&](int w) { return reinterpret_cast<float*>(sm + static_cast<size_t>(w) * kStagesW * 2 * kPageBytes); };

    if (lane == 0) {
        for (int s = 0; s < kStagesW; ++s) mbar_init(&full[warp][s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t pol = l2_evict_first();
    auto issue = [&](int page, int st) {
        const int id = bt[static_cast<int64_t>(s_id) * max_pages + page];
        const int64_t off = (static_cast<int64_t>(id) * nkv + h) * kPageElems;
        uint8_t* dst = ring + st * 2 * kPageBytes;
        mbar_expect_tx(&full[warp][st], 2 * kPageBytes);
        bulk_g2s(dst, kp + off, kPageBytes, &full[warp][st], pol);
        bulk_g2s(dst + kPageBytes, vp + off, kPageBytes, &full[warp][st], pol);
    };
    if (lane == 0)
        for (int k = 0; k < kStagesW && p0 + warp + k * kWarps < n_pages; ++k) issue(p0 + warp + k * kWarps, k);

    // Q^T as B fragments: b0 = q[head g][16kk + 2tg, +1], b1 = q[head g][16kk + 8 + 2tg, +1]
    uint32_t qb[8][2];
    {
        const bool valid = g < G;
        const uint16_t* src = q + static_cast<int64_t>(t) * ldq + (h * G + (valid ? g : 0)) * kD + 2 * tg;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qb[kk][0] = valid ? *reinterpret_cast<const uint32_t*>(src + kk * 16) : 0u;
            qb[kk][1] = valid ? *reinterpret_cast<const uint32_t*>(src + kk * 16 + 8) : 0u;
        }
    }
    const float sl2 = 1.4426950408889634f * rsqrtf(static_cast<float>(kD));
    // this thread's heads: c = 2tg + {0,1}
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

    uint32_t phase = 0;
    for (int k = 0;; ++k) {
        const int page = p0 + warp + k * kWarps;
        if (page >= n_pages) break;
        const int st = k % kStagesW;
        mbar_wait(&full[warp][st], phase);
        const uint32_t sk = ring_s + st * 2 * kPageBytes;
        const uint32_t sv = sk + kPageBytes;
        const int ntok = min(kPage, L - page * kPage);

        page_step(sk, sv, ntok, qb, sl2, lane, m, l, acc);
        __syncwarp();  // every lane is done with this stage
        if (lane == 0 && page + kStagesW * kWarps < n_pages) issue(page + kStagesW * kWarps, st);
        if (st == kStagesW - 1) phase ^= 1;
    }
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) {
        l[0] += __shfl_xor_sync(0xffffffffu, l[0], o);
        l[1] += __shfl_xor_sync(0xffffffffu, l[1], o);
    }

    // ---- merge the warps' partial softmax states: comb[warp][head][d | m | l] ----
    {
        float* cw = comb(warp);  // every copy into this warp's ring has been consumed
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            float* ch = cw + (2 * tg + e) * kCombStride;
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                ch[mt * 16 + g] = acc[mt][e];
                ch[mt * 16 + g + 8] = acc[mt][2 + e];
            }
            if (g == 0) {
                ch[kD] = m[e];
                ch[kD + 1] = l[e];
            }
        }
    }
    __syncthreads();
    // partial of split sp: [t][h][sp][head][O(128) | m | l]
    constexpr int kPart = kD + 2;
    float* const mine = S > 1 ? part + ((static_cast<int64_t>(t) * nkv + h) * S + sp) * (G * kPart) : nullptr;
    for (int idx = threadIdx.x; idx < G * kD; idx += blockDim.x) {
        const int hh = idx / kD, d = idx % kD;
        float M = -INFINITY;
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, comb(w)[hh * kCombStride + kD]);
        float den = 0.f, num = 0.f;
        for (int w = 0; w < kWarps; ++w) {
            const float* c = comb(w) + hh * kCombStride;
            const float f = c[kD + 1] > 0.f ? exp2f(c[kD] - M) : 0.f;  // idle warps: l = 0
            den += c[kD + 1] * f;
            num += c[d] * f;
        }
        if (S > 1) {  // unnormalised partial; the last split merges
            mine[hh * kPart + d] = num;
            if (d == 0) {
                mine[hh * kPart + kD] = M;
                mine[hh * kPart + kD + 1] = den;
            }
            continue;
        }
        const float o = num / den;
        const int col = (h * G + hh) * kD + d;
        if (out_p) *reinterpret_cast<uint16_t*>(out_p + b_packed_off(t, col, R)) = f32_to_bf16_bits(o);
        if (out_f) out_f[static_cast<int64_t>(t) * (G * static_cast<int64_t>(nkv)) * kD + col] = o;
    }
    if (S == 1) return;
    __threadfence();  // this split's partial is visible device-wide before it is counted
    __syncthreads();
    if (threadIdx.x == 0) last_split = atomicAdd(cnt + t * nkv + h, 1) == S - 1;
    __syncthreads();
    if (!last_split) return;
    __threadfence();  // acquire: every other split's partial
    const float* base = part + (static_cast<int64_t>(t) * nkv + h) * S * (G * kPart);
    for (int idx = threadIdx.x; idx < G * kD; idx += blockDim.x) {
        const int hh = idx / kD, d = idx % kD;
        float M = -INFINITY;
        for (int s2 = 0; s2 < S; ++s2) M = fmaxf(M, __ldcg(base + s2 * (G * kPart) + hh * kPart + kD));
        float den = 0.f, num = 0.f;
        for (int s2 = 0; s2 < S; ++s2) {  // split order: deterministic whoever merges
            const float* c = base + s2 * (G * kPart) + hh * kPart;
            const float l2 = __ldcg(c + kD + 1);
            const float f = l2 > 0.f ? exp2f(__ldcg(c + kD) - M) : 0.f;  // empty splits: l = 0
            den += l2 * f;
            num += __ldcg(c + d) * f;
        }
        const float o = num / den;
        const int col = (h * G + hh) * kD + d;
        if (out_p) *reinterpret_cast<uint16_t*>(out_p + b_packed_off(t, col, R)) = f32_to_bf16_bits(o);
        if (out_f) out_f[static_cast<int64_t>(t) * (G * static_cast<int64_t>(nkv)) * kD + col] = o;
    }
    if (threadIdx.x == 0) cnt[t * nkv + h] = 0;  // every split has arrived: ready for the next launch
}

// ---- stream-K decode: the flattened (token, kv head, page) space ----------
// One CTA per (token, kv head) quantises the work: at mu = 64, 8 kv heads,
// 512 equal CTAs are 1.73 waves of the 296 resident slots, and splitting a
// token's pages over extra CTAs (split-KV above) pays each short CTA's
// pipeline ramp and merge.  Here the grid is exactly the resident warps, and
// warp w of W takes the contiguous range [w*P/W, (w+1)*P/W) of the P pages of
// all (token, head) pairs in (token, head, page) order — every warp streams
// the same number of pages with one continuous 3-deep ring across segment
// boundaries.  A (token, head) segment wholly inside a warp's range is
// finished in registers and written out; the (at most two) segments a range
// shares with its neighbours leave a partial (O, m, l) in the warp's slot,
// and the last covering warp to arrive (per-(token, head) counter, reset by
// it) merges the parts in warp order: deterministic for any arrival order.
__device__ __forceinline__ int64_t owner_warp(int64_t s, int64_t W, int64_t P) {  // warp whose range holds s
    return ((s + 1) * W - 1) / P;
}

template <int G>
__global__ void __launch_bounds__(kWarps * 32) gqa_decode_flat_kernel(
    const uint16_t* __restrict__ q, int ldq, const uint16_t* __restrict__ kp, const uint16_t* __restrict__ vp,
    const int32_t* __restrict__ bt, int max_pages, const int32_t* __restrict__ seq, const int32_t* __restrict__ ctx,
    int T, int nkv, uint8_t* out_p, int R, float* out_f, float* __restrict__ part, int* __restrict__ cnt) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[kWarps][kStagesW];
    int* pre = reinterpret_cast<int*>(sm + kWarps * kStagesW * 2 * kPageBytes);  // [T + 1] page prefix
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tg = lane & 3;
    constexpr int kPartF = G * (kD + 2);  // one part: [head][O(128) | m | l]

    // pages per token -> exclusive prefix (block-wide, chunks of blockDim)
    if (threadIdx.x == 0) pre[0] = 0;
    __shared__ int carry_s, wsum[kWarps];
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < T; base += blockDim.x) {
        const int t = base + threadIdx.x;
        int v = t < T ? (ctx[t] + kPage - 1) / kPage : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // inclusive warp scan
            const int n = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += n;
        }
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        int off = carry_s;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        if (t < T) pre[t + 1] = off + v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry_s = off + v;
        __syncthreads();
    }
    const int64_t P = static_cast<int64_t>(nkv) * pre[T];
    // W <= P working warps, so every range is non-empty and the warps covering
    // a segment are exactly owner(s0) .. owner(s1 - 1)
    const int64_t W = min(static_cast<int64_t>(gridDim.x) * kWarps, P);
    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (gw >= W) return;  // no barriers below: idle warps may leave
    const int64_t f0 = gw * P / W, f1 = (gw + 1) * P / W;

    uint8_t* ring = sm + static_cast<size_t>(warp) * kStagesW * 2 * kPageBytes;
    const uint32_t ring_s = smem_u32(ring);
    if (lane == 0) {
        for (int s2 = 0; s2 < kStagesW; ++s2) mbar_init(&full[warp][s2], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // flat page f -> (token, head, page): t = last token with nkv * pre[t] <= f
    auto locate = [&](int64_t f, int& t, int& h, int& p) {
        int lo = 0, hi = T - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (static_cast<int64_t>(nkv) * pre[mid] <= f) lo = mid; else hi = mid - 1;
        }
        t = lo;
        const int np = pre[t + 1] - pre[t];
        const int r = static_cast<int>(f - static_cast<int64_t>(nkv) * pre[t]);
        h = r / np;
        p = r % np;
    };
    const uint64_t pol = l2_evict_first();
    auto issue = [&](int64_t f, int st) {
        int t, h, p;
        locate(f, t, h, p);
        const int id = bt[static_cast<int64_t>(seq[t]) * max_pages + p];
        const int64_t off = (static_cast<int64_t>(id) * nkv + h) * kPageElems;
        uint8_t* dst = ring + st * 2 * kPageBytes;
        mbar_expect_tx(&full[warp][st], 2 * kPageBytes);
        bulk_g2s(dst, kp + off, kPageBytes, &full[warp][st], pol);
        bulk_g2s(dst + kPageBytes, vp + off, kPageBytes, &full[warp][st], pol);
    };
    if (lane == 0)
        for (int k = 0; k < kStagesW && f0 + k < f1; ++k) issue(f0 + k, k);

    const float sl2 = 1.4426950408889634f * rsqrtf(static_cast<float>(kD));
    uint32_t qb[8][2];
    float m[2], l[2], acc[8][4];
    int cur_t = -1, cur_h = -1, L = 0;
    // finish the segment (cur_t, cur_h) whose part of this warp's range ends here
    auto finish = [&]() {
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) {
            l[0] += __shfl_xor_sync(0xffffffffu, l[0], o);
            l[1] += __shfl_xor_sync(0xffffffffu, l[1], o);
        }
        const int np = pre[cur_t + 1] - pre[cur_t];
        const int64_t s0 = static_cast<int64_t>(nkv) * pre[cur_t] + static_cast<int64_t>(cur_h) * np, s1 = s0 + np;
        auto store = [&](int head, int d, float o) {
            const int col = (cur_h * G + head) * kD + d;
            if (out_p) *reinterpret_cast<uint16_t*>(out_p + b_packed_off(cur_t, col, R)) = f32_to_bf16_bits(o);
            if (out_f) out_f[static_cast<int64_t>(cur_t) * (G * static_cast<int64_t>(nkv)) * kD + col] = o;
        };
        if (s0 >= f0 && s1 <= f1) {  // the whole segment is this warp's: normalise in registers
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (2 * tg + e >= G) continue;
                const float inv = 1.0f / l[e];
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    store(2 * tg + e, mt * 16 + g, acc[mt][e] * inv);
                    store(2 * tg + e, mt * 16 + g + 8, acc[mt][2 + e] * inv);
                }
            }
            return;
        }
        // shared segment: this warp's part -> its slot (0: the range's first segment, 1: its last)
        const int slot = s0 < f0 ? 0 : 1;
        float* mine = part + (gw * 2 + slot) * kPartF;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (2 * tg + e >= G) continue;
            float* ph = mine + (2 * tg + e) * (kD + 2);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                ph[mt * 16 + g] = acc[mt][e];
                ph[mt * 16 + g + 8] = acc[mt][2 + e];
            }
            if (g == 0) {
                ph[kD] = m[e];
                ph[kD + 1] = l[e];
            }
        }
        __threadfence();
        __syncwarp();
        const int64_t w_first = owner_warp(s0, W, P), w_last = owner_warp(s1 - 1, W, P);
        const int nparts = static_cast<int>(w_last - w_first + 1);
        int last = 0;
        if (lane == 0) last = atomicAdd(cnt + cur_t * nkv + cur_h, 1) == nparts - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) return;
        __threadfence();  // acquire the other parts
        // merge in warp order (deterministic), 8 parts at a time with every
        // load of a batch in flight before the arithmetic (one L2 round trip
        // per batch and head instead of one per part)
        auto slot_of = [&](int64_t w) { return s0 < w * P / W ? 0 : 1; };  // as the writer chose
        for (int hh = 0; hh < G; ++hh) {
            float M = -INFINITY, den = 0.f, num[4] = {0.f, 0.f, 0.f, 0.f};
            for (int64_t w0 = w_first; w0 <= w_last; w0 += 8) {
                float mv[8], lv[8], ov[8][4];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int64_t w = w0 + j;
                    if (w <= w_last) {
                        const float* c = part + (w * 2 + slot_of(w)) * kPartF + hh * (kD + 2);
                        mv[j] = __ldcg(c + kD);
                        lv[j] = __ldcg(c + kD + 1);
#pragma unroll
                        for (int i = 0; i < 4; ++i) ov[j][i] = __ldcg(c + lane + 32 * i);
                    } else {
                        mv[j] = -INFINITY;
                        lv[j] = 0.f;
#pragma unroll
                        for (int i = 0; i < 4; ++i) ov[j][i] = 0.f;
                    }
                }
                float Mn = M;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (lv[j] > 0.f) Mn = fmaxf(Mn, mv[j]);
                const float sc = den > 0.f ? exp2f(M - Mn) : 0.f;  // rescale what is merged so far
                den *= sc;
#pragma unroll
                for (int i = 0; i < 4; ++i) num[i] *= sc;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float f = lv[j] > 0.f ? exp2f(mv[j] - Mn) : 0.f;
                    den += lv[j] * f;
#pragma unroll
                    for (int i = 0; i < 4; ++i) num[i] += ov[j][i] * f;
                }
                M = Mn;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) store(hh, lane + 32 * i, num[i] / den);
        }
        if (lane == 0) cnt[cur_t * nkv + cur_h] = 0;
    };

    uint32_t phase = 0;
    for (int64_t k = 0; f0 + k < f1; ++k) {
        const int st = static_cast<int>(k % kStagesW);
        int t, h, p;
        locate(f0 + k, t, h, p);
        if (t != cur_t || h != cur_h) {
            if (cur_t >= 0) finish();
            cur_t = t;
            cur_h = h;
            L = ctx[t];
            const bool valid = g < G;
            const uint16_t* src = q + static_cast<int64_t>(t) * ldq + (h * G + (valid ? g : 0)) * kD + 2 * tg;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                qb[kk][0] = valid ? *reinterpret_cast<const uint32_t*>(src + kk * 16) : 0u;
                qb[kk][1] = valid ? *reinterpret_cast<const uint32_t*>(src + kk * 16 + 8) : 0u;
            }
            m[0] = m[1] = -INFINITY;
            l[0] = l[1] = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
        }
        mbar_wait(&full[warp][st], phase);
        const uint32_t sk = ring_s + st * 2 * kPageBytes;
        page_step(sk, sk + kPageBytes, min(kPage, L - p * kPage), qb, sl2, lane, m, l, acc);
        __syncwarp();  // every lane is done with this stage
        if (lane == 0 && f0 + k + kStagesW < f1) issue(f0 + k + kStagesW, st);
        if (st == kStagesW - 1) phase ^= 1;
    }
    finish();
}

// One CTA per token: 16-byte chunks of this step's K and V rows into the
// swizzled page slot of position pos[t].
__global__ void kv_append_kernel(const uint16_t* qkv, int nq, int nkv, int d, const int32_t* seq,
                                 const int32_t* pos, const int32_t* bt, int max_pages, int page,
                                 uint16_t* kp, uint16_t* vp) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    const int t = blockIdx.x;
    const int W = (nq + 2 * nkv) * d;
    const int p = pos[t];
    const int id = bt[static_cast<int64_t>(seq[t]) * max_pages + p / page];
    const int within = p % page;
    const int cpr = d / 8;
    for (int j = threadIdx.x; j < 2 * nkv * cpr; j += blockDim.x) {
        const int which = j / (nkv * cpr), jj = j % (nkv * cpr);
        const int hh = jj / cpr, c = jj % cpr;
        const int64_t off = (static_cast<int64_t>(id) * nkv + hh) * page * d + kv_page_off(within, c * 8);
        const uint4 v = *reinterpret_cast<const uint4*>(qkv + static_cast<int64_t>(t) * W + (nq + which * nkv) * d + jj * 8);
        *reinterpret_cast<uint4*>((which ? vp : kp) + off) = v;
    }
}
template <int G>
cudaError_t launch_g(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp,
                     const int32_t* bt, int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                     int nkv, uint8_t* out_p, int R, float* out_f, const GqaSplit* split, cudaStream_t s) {
    const int smem = kWarps * kStagesW * 2 * kPageBytes;
    static_assert(8 * kCombStride * 4 <= kStagesW * 2 * kPageBytes, "merge state fits a warp's ring");
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gqa_decode_kernel<G>), smem); e != cudaSuccess)
        return e;
    int S = 1;
    if (split && split->scratch && split->counters) {
        S = split->splits;
        if (S <= 0) {  // auto: the split count in 1..max whose grid best fills whole waves, keeping
                       // >= kMinSplitPages pages per split (a split CTA pays its pipeline ramp and
                       // merge once: 8-page splits measured 2x slower at mu = 64, ctx 528)
            // resident-CTA slots of this device, cached (the occupancy query costs
            // microseconds of host time per call)
            static int cache_slots[64] = {};
            int dev = 0;
            if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidValue;
            if (!cache_slots[dev]) {
                int per_sm = 0, sms = 0;
                if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gqa_decode_kernel<G>, kWarps * 32, smem) !=
                        cudaSuccess)
                    return cudaErrorInvalidValue;
                cache_slots[dev] = sms * (per_sm > 0 ? per_sm : 1);
            }
            const int per_sm = 1, sms = cache_slots[dev];
            const double slots = static_cast<double>(sms) * (per_sm > 0 ? per_sm : 1);
            double best = 0;
            for (int c = 1; c <= split->max_splits && max_pages / c >= kMinSplitPages; ++c) {
                const double w = static_cast<double>(T) * nkv * c / slots;
                const double fill = w / std::ceil(w);
                if (fill > best + 0.02) best = fill, S = c;  // more splits only for a clearly better fill
            }
        }
        if (S > split->max_splits) return cudaErrorInvalidValue;
    }
    if (S < 1) S = 1;
    dim3 grid(T, nkv, S);
    return launch_k(gqa_decode_kernel<G>, dim3(grid), dim3(kWarps * 32), smem, s, q, ldq, kp, vp, bt, max_pages, seq, ctx, nkv,
                    out_p, R, out_f, S, S > 1 ? split->scratch : nullptr, S > 1 ? split->counters : nullptr);
}

template <int G>
cudaError_t launch_flat(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp, const int32_t* bt,
                        int max_pages, const int32_t* seq, const int32_t* ctx, int T, int nkv, uint8_t* out_p, int R,
                        float* out_f, const GqaFlat& fl, cudaStream_t s) {
    const int smem = kWarps * kStagesW * 2 * kPageBytes + (T + 1) * 4;
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gqa_decode_flat_kernel<G>),
                                         kWarps * kStagesW * 2 * kPageBytes + (kMaxFlatTokens + 1) * 4);
        e != cudaSuccess)
        return e;
    return launch_k(gqa_decode_flat_kernel<G>, dim3(fl.ctas), dim3(kWarps * 32), smem, s, q, ldq, kp, vp, bt, max_pages,
                    seq, ctx, T, nkv, out_p, R, out_f, fl.scratch, fl.counters);
}

}  // namespace

int gqa_flat_ctas(int num_sms) { return 2 * num_sms; }  // 96 KiB rings: 2 CTAs per SM

cudaError_t launch_gqa_decode_flat(const uint16_t* q, int ldq, const uint16_t* k_pool, const uint16_t* v_pool,
                                   const int32_t* block_table, int max_pages, const int32_t* seq, const int32_t* ctx,
                                   int T, int nq, int nkv, int d, int page, uint8_t* out_packed, int R,
                                   float* out_rowmajor, const GqaFlat& fl, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (d != kD || nq % nkv || page != kPage || T > kMaxFlatTokens || fl.ctas < 1 || !fl.scratch || !fl.counters)
        return cudaErrorInvalidValue;
    switch (nq / nkv) {
        case 1: return launch_flat<1>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, fl, s);
        case 2: return launch_flat<2>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, fl, s);
        case 4: return launch_flat<4>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, fl, s);
        case 6: return launch_flat<6>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, fl, s);
        case 8: return launch_flat<8>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, fl, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gqa_decode_paged(const uint16_t* q, int ldq, const uint16_t* k_pool,
                                    const uint16_t* v_pool, const int32_t* block_table,
                                    int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                                    int nq, int nkv, int d, int page, uint8_t* out_packed, int R,
                                    float* out_rowmajor, cudaStream_t s, const GqaSplit* split) {
    if (T <= 0) return cudaSuccess;
    if (d != kD || nq % nkv || page != kPage) return cudaErrorInvalidValue;
    switch (nq / nkv) {
        case 1: return launch_g<1>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, split, s);
        case 2: return launch_g<2>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, split, s);
        case 4: return launch_g<4>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, split, s);
        case 6: return launch_g<6>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, split, s);
        case 8: return launch_g<8>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, split, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_kv_append(const uint16_t* qkv_bf16, int nq, int nkv, int d, const int32_t* seq,
                             const int32_t* pos, int T, const int32_t* block_table, int max_pages,
                             int page, uint16_t* k_pool, uint16_t* v_pool, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    return launch_k(kv_append_kernel, dim3(T), dim3(256), 0, s, qkv_bf16, nq, nkv, d, seq, pos, block_table, max_pages,
                                       page, k_pool, v_pool);
}

}  // namespace mltk
