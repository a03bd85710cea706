// GQA decode attention over a paged KV cache (north_star item 4; SURVEY.md
// §2c gqa_decode_paged), used when the policy places attention on the GPU
// (A_g = 1).  Memory-bound: attention intensity is 2*n_q/(n_kv*dt_kv) FLOP/B
// (4 for 8x7B), so the kernel's job is to stream K/V pages at HBM rate.
//
// Layout: a KV page holds kPage = 16 consecutive tokens of ONE kv head,
// [16][d] bf16 (K and V in separate pools), so a (page, head) slice is one
// contiguous 4 KiB run that a single cp.async.bulk moves into shared memory.
// Page id = block_table[seq][pos / 16]; pool offset = (id*n_kv + h)*16*d.
//
// One CTA per (query token, kv head).  Its kWarps warps split the pages
// (warp w takes pages w, w+kWarps, ...: flash-decoding inside the CTA) and
// each warp serves ALL G = n_q/n_kv query heads of the kv head, so every
// K/V element is read once from HBM and once from shared memory for all G
// heads (GQA reuse).  Each warp owns a kStagesW-deep ring of pages that its
// lane 0 fills with 1-D bulk copies (mbarrier tx counts): the page gather is
// staged through shared memory, ahead of the math.
//   QK^T: 8 lanes per token (16 dims each, q in registers pre-scaled by
//         log2(e)/sqrt(d)), 4 tokens per pass; lanes of the upper half read
//         their two 16-byte chunks in swapped order so a pass is
//         bank-conflict-free; 3 xor-shuffles reduce a score.
//   softmax: exp2 domain, one 2-shuffle warp max/sum per page and head.
//   PV: lane l owns dims [4l, 4l+4); p_j arrives by shuffle.
// The warps' (m, l, acc) are merged through shared memory at the end.
#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kPage = 16;
constexpr int kD = 128;
constexpr int kWarps = 4;
constexpr int kStagesW = 3;
constexpr int kPageElems = kPage * kD;
constexpr int kPageBytes = kPageElems * 2;  // 4 KiB (one of K or V)
constexpr int kCombStride = 4 + kD;         // [m, l, pad, pad, acc[128]]: 16-byte aligned rows

__device__ __forceinline__ float lo_bf16(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float hi_bf16(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

template <int G>
__global__ void __launch_bounds__(kWarps * 32) gqa_decode_kernel(
    const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp, const int32_t* bt,
    int max_pages, const int32_t* seq, const int32_t* ctx, int nkv, uint8_t* out_p, int R,
    float* out_f) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[kWarps][kStagesW];
    const int t = blockIdx.x, h = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = ctx[t];
    const int s_id = seq[t];
    const int n_pages = (L + kPage - 1) / kPage;
    // per-warp ring: [warp][stage][K page | V page]
    uint16_t* ring = reinterpret_cast<uint16_t*>(sm) + static_cast<size_t>(warp) * kStagesW * 2 * kPageElems;
    float* comb = reinterpret_cast<float*>(sm + kWarps * kStagesW * 2 * kPageBytes);  // [warp][G][2 + kD]

    if (lane == 0) {
        for (int s = 0; s < kStagesW; ++s) mbar_init(&full[warp][s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t pol = l2_evict_first();
    auto issue = [&](int page, int st) {
        const int id = bt[static_cast<int64_t>(s_id) * max_pages + page];
        const int64_t off = (static_cast<int64_t>(id) * nkv + h) * kPageElems;
        uint16_t* dst = ring + st * 2 * kPageElems;
        mbar_expect_tx(&full[warp][st], 2 * kPageBytes);
        bulk_g2s(dst, kp + off, kPageBytes, &full[warp][st], pol);
        bulk_g2s(dst + kPageElems, vp + off, kPageBytes, &full[warp][st], pol);
    };
    if (lane == 0)
        for (int k = 0; k < kStagesW && warp + k * kWarps < n_pages; ++k) issue(warp + k * kWarps, k);

    // q slice: lane (grp = lane/8, r = lane%8) holds dims [16r, 16r+16) of each head
    const int grp = lane >> 3, r = lane & 7;
    const bool swap = (r >> 2) & 1;  // upper half reads its two chunks in swapped order
    const float qscale = 1.4426950408889634f * rsqrtf(static_cast<float>(kD));
    float qr[G][16];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const uint16_t* src = q + static_cast<int64_t>(t) * ldq + (h * G + g) * kD + r * 16;
        const uint4 a = *reinterpret_cast<const uint4*>(src);
        const uint4 b = *reinterpret_cast<const uint4*>(src + 8);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            qr[g][2 * e] = lo_bf16(w[e]) * qscale;
            qr[g][2 * e + 1] = hi_bf16(w[e]) * qscale;
        }
    }
    float m[G], l[G], acc[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = -FLT_MAX;
        l[g] = 0.f;
        acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
    }

    uint32_t phase = 0;
    for (int k = 0;; ++k) {
        const int page = warp + k * kWarps;
        if (page >= n_pages) break;
        const int st = k % kStagesW;
        mbar_wait(&full[warp][st], phase);
        const uint16_t* sk = ring + st * 2 * kPageElems;
        const uint16_t* sv = sk + kPageElems;
        const int ntok = min(kPage, L - page * kPage);

        // ---- QK^T: 4 passes x 4 tokens, 8 lanes per token ----
        float sc[G][4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int tok = p * 4 + grp;
            const uint16_t* row = sk + tok * kD + r * 16;
            float part[G];
#pragma unroll
            for (int g = 0; g < G; ++g) part[g] = 0.f;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int cc = swap ? (c ^ 1) : c;
                const uint4 kv = *reinterpret_cast<const uint4*>(row + cc * 8);
                const uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float q0 = swap ? qr[g][(c ^ 1) * 8 + 2 * e] : qr[g][c * 8 + 2 * e];
                        const float q1 = swap ? qr[g][(c ^ 1) * 8 + 2 * e + 1] : qr[g][c * 8 + 2 * e + 1];
                        part[g] = fmaf(q0, lo_bf16(w[e]), part[g]);
                        part[g] = fmaf(q1, hi_bf16(w[e]), part[g]);
                    }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float v = part[g];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                sc[g][p] = tok < ntok ? v : -FLT_MAX;
            }
        }
        // ---- online softmax per head (exp2 domain) ----
        float pe[G][4];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float tmax = fmaxf(fmaxf(sc[g][0], sc[g][1]), fmaxf(sc[g][2], sc[g][3]));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
            const float m_new = fmaxf(m[g], tmax);
            const float corr = exp2f(m[g] - m_new);
            float ps = 0.f;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                pe[g][p] = (p * 4 + grp) < ntok ? exp2f(sc[g][p] - m_new) : 0.f;
                ps += pe[g][p];
            }
            ps += __shfl_xor_sync(0xffffffffu, ps, 8);
            ps += __shfl_xor_sync(0xffffffffu, ps, 16);
            l[g] = l[g] * corr + ps;
            m[g] = m_new;
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[g][e] *= corr;
        }
        // ---- PV: lane owns dims [4*lane, 4*lane + 4) ----
#pragma unroll
        for (int tok = 0; tok < kPage; ++tok) {
            const uint2 vv = *reinterpret_cast<const uint2*>(sv + tok * kD + lane * 4);
            const float v0 = lo_bf16(vv.x), v1 = hi_bf16(vv.x), v2 = lo_bf16(vv.y), v3 = hi_bf16(vv.y);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float pj = __shfl_sync(0xffffffffu, pe[g][tok >> 2], (tok & 3) * 8);
                acc[g][0] = fmaf(pj, v0, acc[g][0]);
                acc[g][1] = fmaf(pj, v1, acc[g][1]);
                acc[g][2] = fmaf(pj, v2, acc[g][2]);
                acc[g][3] = fmaf(pj, v3, acc[g][3]);
            }
        }
        __syncwarp();  // every lane is done with this stage
        if (lane == 0 && page + kStagesW * kWarps < n_pages) issue(page + kStagesW * kWarps, st);
        if (st == kStagesW - 1) phase ^= 1;
    }

    // ---- merge the warps' partial softmax states ----
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float* c = comb + (warp * G + g) * kCombStride;
        if (lane == 0) {
            c[0] = m[g];
            c[1] = l[g];
        }
        *reinterpret_cast<float4*>(c + 4 + lane * 4) = make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < G * kD; idx += blockDim.x) {
        const int g = idx / kD, d = idx % kD;
        float M = -FLT_MAX;
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, comb[(w * G + g) * kCombStride]);
        float den = 0.f, num = 0.f;
        for (int w = 0; w < kWarps; ++w) {
            const float* c = comb + (w * G + g) * kCombStride;
            const float f = c[1] > 0.f ? exp2f(c[0] - M) : 0.f;
            den += c[1] * f;
            num += c[4 + d] * f;
        }
        const float o = num / den;
        const int col = (h * G + g) * kD + d;
        if (out_p) *reinterpret_cast<uint16_t*>(out_p + b_packed_off(t, col, R)) = f32_to_bf16_bits(o);
        if (out_f) out_f[static_cast<int64_t>(t) * (G * static_cast<int64_t>(nkv)) * kD + col] = o;
    }
}

__global__ void kv_append_kernel(const uint16_t* qkv, int nq, int nkv, int d, const int32_t* seq,
                                 const int32_t* pos, const int32_t* bt, int max_pages, int page,
                                 uint16_t* kp, uint16_t* vp) {
    const int t = blockIdx.x;
    const int W = (nq + 2 * nkv) * d;
    const int p = pos[t];
    const int id = bt[static_cast<int64_t>(seq[t]) * max_pages + p / page];
    const int within = p % page;
    for (int j = threadIdx.x; j < nkv * d; j += blockDim.x) {
        const int h = j / d, i = j % d;
        const int64_t off = ((static_cast<int64_t>(id) * nkv + h) * page + within) * d + i;
        kp[off] = qkv[static_cast<int64_t>(t) * W + nq * d + j];
        vp[off] = qkv[static_cast<int64_t>(t) * W + (nq + nkv) * d + j];
    }
}

template <int G>
cudaError_t launch_g(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp,
                     const int32_t* bt, int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                     int nkv, uint8_t* out_p, int R, float* out_f, cudaStream_t s) {
    const int smem = kWarps * kStagesW * 2 * kPageBytes + kWarps * G * kCombStride * 4;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gqa_decode_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid(T, nkv);
    gqa_decode_kernel<G><<<grid, kWarps * 32, smem, s>>>(q, ldq, kp, vp, bt, max_pages, seq, ctx, nkv,
                                                         out_p, R, out_f);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gqa_decode_paged(const uint16_t* q, int ldq, const uint16_t* k_pool,
                                    const uint16_t* v_pool, const int32_t* block_table,
                                    int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                                    int nq, int nkv, int d, int page, uint8_t* out_packed, int R,
                                    float* out_rowmajor, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (d != kD || nq % nkv || page != kPage) return cudaErrorInvalidValue;
    switch (nq / nkv) {
        case 1: return launch_g<1>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, s);
        case 2: return launch_g<2>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, s);
        case 4: return launch_g<4>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, s);
        case 6: return launch_g<6>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, s);
        case 8: return launch_g<8>(q, ldq, k_pool, v_pool, block_table, max_pages, seq, ctx, T, nkv, out_packed, R, out_rowmajor, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_kv_append(const uint16_t* qkv_bf16, int nq, int nkv, int d, const int32_t* seq,
                             const int32_t* pos, int T, const int32_t* block_table, int max_pages,
                             int page, uint16_t* k_pool, uint16_t* v_pool, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    kv_append_kernel<<<T, 256, 0, s>>>(qkv_bf16, nq, nkv, d, seq, pos, block_table, max_pages,
                                       page, k_pool, v_pool);
    return cudaGetLastError();
}

}  // namespace mltk
