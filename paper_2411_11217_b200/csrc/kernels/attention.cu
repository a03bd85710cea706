// GQA decode attention over a paged KV cache (north_star item 4; SURVEY.md
// §2c gqa_decode_paged), used when the policy places attention on the GPU
// (A_g = 1).  Memory-bound: attention intensity is 2*n_q/(n_kv*dt_kv) FLOP/B
// (4 for 8x7B), so the kernel's job is to stream K/V pages at HBM rate.
//
// Layout: a KV page holds `page` consecutive tokens of ONE kv head,
// [page][d] bf16 (K and V in separate pools), so a (page, head) slice is one
// contiguous run that a single cp.async.bulk moves into shared memory.
// Page id = block_table[seq][pos / page]; pool offset = (id*n_kv + h)*page*d.
//
// One CTA per (query token, kv head): its G = n_q/n_kv query heads share
// every K/V page (GQA reuse).  Warp w handles query head h*G + w; lane l owns
// dims [4l, 4l+4) (d = 128).  Thread 0 keeps a ring of kStages pages in
// flight (mbarrier full/empty), so the page gather is staged through shared
// memory and overlapped with the dot products.  Online softmax per page.
#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kStages = 4;
constexpr int kPage = 16;  // tokens per KV page (compile-time: scores stay in registers)

template <int D>
__global__ void gqa_decode_kernel(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp,
                                  const int32_t* bt, int max_pages, const int32_t* seq,
                                  const int32_t* ctx, int nq, int nkv, int page, uint8_t* out_p,
                                  int R, float* out_f) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[kStages], empty[kStages];
    const int t = blockIdx.x, h = blockIdx.y;
    const int G = nq / nkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = ctx[t];
    const int s_id = seq[t];
    const int n_pages = (L + page - 1) / page;
    const int page_bytes = page * D * 2;
    uint16_t* sk = reinterpret_cast<uint16_t*>(sm);
    uint16_t* sv = reinterpret_cast<uint16_t*>(sm + kStages * page_bytes);
    const int nw = blockDim.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nw);
        }
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int p) {
        const int st = p % kStages;
        const int id = bt[static_cast<int64_t>(s_id) * max_pages + p];
        const int64_t off = (static_cast<int64_t>(id) * nkv + h) * page * D;
        mbar_expect_tx(&full[st], 2 * page_bytes);
        const uint64_t pol = l2_evict_first();
        bulk_g2s(sk + st * page * D, kp + off, page_bytes, &full[st], pol);
        bulk_g2s(sv + st * page * D, vp + off, page_bytes, &full[st], pol);
    };
    if (threadIdx.x == 0)
        for (int p = 0; p < n_pages && p < kStages; ++p) issue(p);

    const int qh = h * G + warp;
    const bool active = warp < G;
    float qv[4] = {0.f, 0.f, 0.f, 0.f};
    if (active) {
        const uint2 raw = *reinterpret_cast<const uint2*>(q + static_cast<int64_t>(t) * ldq + qh * D + lane * 4);
        const uint16_t* b = reinterpret_cast<const uint16_t*>(&raw);
        const float scale = rsqrtf(static_cast<float>(D));
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = bf16_bits_to_f32(b[i]) * scale;
    }
    float m = -FLT_MAX, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t phase = 0;
    for (int p = 0; p < n_pages; ++p) {
        const int st = p % kStages;
        mbar_wait(&full[st], phase);
        const int ntok = min(page, L - p * page);
        if (active) {
            float sc[kPage];
            float pmax = -FLT_MAX;
#pragma unroll
            for (int j = 0; j < kPage; ++j) {
                if (j >= ntok) { sc[j] = -FLT_MAX; continue; }
                const uint2 raw = *reinterpret_cast<const uint2*>(sk + (st * page + j) * D + lane * 4);
                const uint16_t* b = reinterpret_cast<const uint16_t*>(&raw);
                float s = qv[0] * bf16_bits_to_f32(b[0]) + qv[1] * bf16_bits_to_f32(b[1]) +
                          qv[2] * bf16_bits_to_f32(b[2]) + qv[3] * bf16_bits_to_f32(b[3]);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                sc[j] = s;
                pmax = fmaxf(pmax, s);
            }
            const float m_new = fmaxf(m, pmax);
            const float corr = __expf(m - m_new);
            l *= corr;
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] *= corr;
#pragma unroll
            for (int j = 0; j < kPage; ++j) {
                if (j >= ntok) continue;
                const float pj = __expf(sc[j] - m_new);
                l += pj;
                const uint2 raw = *reinterpret_cast<const uint2*>(sv + (st * page + j) * D + lane * 4);
                const uint16_t* b = reinterpret_cast<const uint16_t*>(&raw);
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[i] += pj * bf16_bits_to_f32(b[i]);
            }
            m = m_new;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (threadIdx.x == 0 && p + kStages < n_pages) {
            mbar_wait(&empty[st], phase);
            issue(p + kStages);
        }
        if (st == kStages - 1) phase ^= 1;
    }
    if (active) {
        const float inv = L > 0 ? 1.0f / l : 0.0f;
        const int col = qh * D + lane * 4;
        uint2 o;
        uint16_t* ob = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
        for (int i = 0; i < 4; ++i) ob[i] = f32_to_bf16_bits(acc[i] * inv);
        if (out_p) *reinterpret_cast<uint2*>(out_p + b_packed_off(t, col, R)) = o;
        if (out_f)
            *reinterpret_cast<float4*>(out_f + static_cast<int64_t>(t) * nq * D + col) =
                make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
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

}  // namespace

cudaError_t launch_gqa_decode_paged(const uint16_t* q, int ldq, const uint16_t* k_pool,
                                    const uint16_t* v_pool, const int32_t* block_table,
                                    int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                                    int nq, int nkv, int d, int page, uint8_t* out_packed, int R,
                                    float* out_rowmajor, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (d != 128 || nq % nkv || nq / nkv > 32 || page != kPage)
        return cudaErrorInvalidValue;
    const int G = nq / nkv;
    const int threads = ((G + 0) * 32 < 64) ? 64 : G * 32;
    const int smem = 2 * kStages * page * d * 2;
    dim3 grid(T, nkv);
    gqa_decode_kernel<128><<<grid, threads, smem, s>>>(q, ldq, k_pool, v_pool, block_table, max_pages,
                                                       seq, ctx, nq, nkv, page, out_packed, R,
                                                       out_rowmajor);
    return cudaGetLastError();
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
