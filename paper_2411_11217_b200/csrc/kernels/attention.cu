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
// One CTA per (query token, kv head); warp g handles query head h*G + g, so
// every K/V tile is read from HBM once for all G heads (GQA reuse).  Tiles of
// 32 tokens (two pages of K and V, 16 KiB) flow through a kStages-deep ring
// filled by one elected thread with 1-D bulk copies (mbarrier tx counts) —
// the page gather is staged through shared memory.  QK^T: lane j owns token
// j of the tile and walks the 128 dims in 16-byte chunks rotated by j
// (conflict-free), against q held in shared memory pre-scaled by
// log2(e)/sqrt(d); softmax runs in the exp2 domain with one warp max/sum per
// tile; PV: lane l owns dims [4l, 4l+4) and takes p_j by shuffle.
#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kPage = 16;
constexpr int kTile = 32;          // tokens per tile (2 pages)
constexpr int kD = 128;
constexpr int kStages = 4;
constexpr int kTileBytes = kTile * kD * 2;  // one of K or V: 8 KiB

__global__ void __launch_bounds__(256) gqa_decode_kernel(const uint16_t* q, int ldq, const uint16_t* kp,
                                                          const uint16_t* vp, const int32_t* bt,
                                                          int max_pages, const int32_t* seq,
                                                          const int32_t* ctx, int nq, int nkv,
                                                          uint8_t* out_p, int R, float* out_f) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[kStages], empty[kStages];
    const int t = blockIdx.x, h = blockIdx.y;
    const int G = nq / nkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = ctx[t];
    const int s_id = seq[t];
    const int n_pages = (L + kPage - 1) / kPage;
    const int n_tiles = (L + kTile - 1) / kTile;
    uint16_t* sk = reinterpret_cast<uint16_t*>(sm);                               // [stages][32][128]
    uint16_t* sv = reinterpret_cast<uint16_t*>(sm + kStages * kTileBytes);        // [stages][32][128]
    float* sq = reinterpret_cast<float*>(sm + 2 * kStages * kTileBytes);          // [G][128]

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G);
        }
        fence_mbar_init();
    }
    // q for the G heads of this kv head, fp32, pre-scaled for exp2-domain softmax
    const float qscale = 1.4426950408889634f * rsqrtf(static_cast<float>(kD));
    for (int i = threadIdx.x; i < G * kD; i += blockDim.x)
        sq[i] = bf16_bits_to_f32(q[static_cast<int64_t>(t) * ldq + (h * G) * kD + i]) * qscale;
    __syncthreads();

    const uint64_t pol = l2_evict_first();
    auto issue = [&](int tile) {
        const int st = tile % kStages;
        const int p0 = tile * 2;
        const int np = min(2, n_pages - p0);
        mbar_expect_tx(&full[st], np * 2 * kPage * kD * 2);
        for (int i = 0; i < np; ++i) {
            const int id = bt[static_cast<int64_t>(s_id) * max_pages + p0 + i];
            const int64_t off = (static_cast<int64_t>(id) * nkv + h) * kPage * kD;
            bulk_g2s(sk + (st * kTile + i * kPage) * kD, kp + off, kPage * kD * 2, &full[st], pol);
            bulk_g2s(sv + (st * kTile + i * kPage) * kD, vp + off, kPage * kD * 2, &full[st], pol);
        }
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < n_tiles && i < kStages; ++i) issue(i);

    const bool active = warp < G;
    const float* qg = sq + warp * kD;
    float m = -FLT_MAX, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t phase = 0;
    for (int i = 0; i < n_tiles; ++i) {
        const int st = i % kStages;
        mbar_wait(&full[st], phase);
        const int ntok = min(kTile, L - i * kTile);
        if (active) {
            // ---- scores: lane j <-> token j ----
            float s = -FLT_MAX;
            if (lane < ntok) {
                const uint16_t* krow = sk + (st * kTile + lane) * kD;
                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                for (int c = 0; c < kD / 8; ++c) {
                    const int cr = (c + lane) & (kD / 8 - 1);
                    const uint4 kv = *reinterpret_cast<const uint4*>(krow + cr * 8);
                    const float4 qa = *reinterpret_cast<const float4*>(qg + cr * 8);
                    const float4 qb = *reinterpret_cast<const float4*>(qg + cr * 8 + 4);
                    a0 = fmaf(qa.x, __uint_as_float(kv.x << 16), a0);
                    a1 = fmaf(qa.y, __uint_as_float(kv.x & 0xffff0000u), a1);
                    a0 = fmaf(qa.z, __uint_as_float(kv.y << 16), a0);
                    a1 = fmaf(qa.w, __uint_as_float(kv.y & 0xffff0000u), a1);
                    a0 = fmaf(qb.x, __uint_as_float(kv.z << 16), a0);
                    a1 = fmaf(qb.y, __uint_as_float(kv.z & 0xffff0000u), a1);
                    a0 = fmaf(qb.z, __uint_as_float(kv.w << 16), a0);
                    a1 = fmaf(qb.w, __uint_as_float(kv.w & 0xffff0000u), a1);
                }
                s = a0 + a1;
            }
            // ---- online softmax (exp2 domain), one warp reduction per tile ----
            float tmax = s;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            const float m_new = fmaxf(m, tmax);
            const float corr = exp2f(m - m_new);
            const float p = lane < ntok ? exp2f(s - m_new) : 0.f;
            float psum = p;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
            l = l * corr + psum;
            m = m_new;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] *= corr;
            // ---- PV: lane l <-> dims [4l, 4l+4) ----
            const uint16_t* vbase = sv + st * kTile * kD + lane * 4;
#pragma unroll 8
            for (int j = 0; j < kTile; ++j) {
                const float pj = __shfl_sync(0xffffffffu, p, j);
                const uint2 vv = *reinterpret_cast<const uint2*>(vbase + j * kD);
                acc[0] = fmaf(pj, __uint_as_float(vv.x << 16), acc[0]);
                acc[1] = fmaf(pj, __uint_as_float(vv.x & 0xffff0000u), acc[1]);
                acc[2] = fmaf(pj, __uint_as_float(vv.y << 16), acc[2]);
                acc[3] = fmaf(pj, __uint_as_float(vv.y & 0xffff0000u), acc[3]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (threadIdx.x == 0 && i + kStages < n_tiles) {
            mbar_wait(&empty[st], phase);
            issue(i + kStages);
        }
        if (st == kStages - 1) phase ^= 1;
    }
    if (active) {
        const float inv = 1.0f / l;
        const int col = (h * G + warp) * kD + lane * 4;
        uint2 o;
        uint16_t* ob = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) ob[k] = f32_to_bf16_bits(acc[k] * inv);
        if (out_p) *reinterpret_cast<uint2*>(out_p + b_packed_off(t, col, R)) = o;
        if (out_f)
            *reinterpret_cast<float4*>(out_f + static_cast<int64_t>(t) * nq * kD + col) =
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
    if (d != kD || nq % nkv || nq / nkv > 8 || page != kPage) return cudaErrorInvalidValue;
    const int G = nq / nkv;
    const int threads = G * 32;
    const int smem = 2 * kStages * kTileBytes + G * kD * 4;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gqa_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             2 * kStages * kTileBytes + 8 * kD * 4);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid(T, nkv);
    gqa_decode_kernel<<<grid, threads, smem, s>>>(q, ldq, k_pool, v_pool, block_table, max_pages, seq,
                                                  ctx, nq, nkv, out_packed, R, out_rowmajor);
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
