// Top-k router + token permutation (north_star item 2; SURVEY.md §2c
// router_topk_permute), warp-level.
//
// router_kernel: one CTA (H/8 threads) per token.  Optional fused RMSNorm of the fp32
// residual (the PostAttn norm), then one warp per expert computes the logit
// with the FIXED reduction tree of oracle/oracle_numerics.c:orc_router —
// lane l accumulates 8-element chunks c = l, l+32, ... with fmaf in element
// order, then a xor butterfly 16,8,4,2,1 — so on identical bf16 inputs the
// logits, the top-k indices and the permutation are bit-identical to the CPU
// oracle.  Top-k on logits (softmax is monotone), ties to the lower index;
// weights = softmax over the k selected logits.
//
// permute_kernel: every CTA recomputes the stable (expert, token, slot)
// order from topk_idx with warp ballots (no atomics -> deterministic), pads
// each expert segment to 16 rows (UMMA N granularity), and gathers its share
// of hn rows into the packed expert operand.  CTA 0 publishes counts,
// offsets, perm and inv.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kMaxE = 64;
constexpr int kMaxSlots = 16384;  // T*K per launch (prefill chunks)

// One CTA of H/8 threads per token; thread i owns elements [8i, 8i+8) and
// issues every load of its slice (split-K partials + residual) up front.
__global__ void __launch_bounds__(768) router_kernel(const float* x, const uint16_t* gamma, float eps,
                                                      const uint16_t* hn_in, const uint16_t* w, int H, int E,
                                                      int K, uint16_t* hn_out, float* logits, int32_t* topk_idx,
                                                      float* topk_w, int parts, int64_t part_stride,
                                                      const float* residual, float* h_out) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    extern __shared__ __align__(16) uint8_t sm[];
    uint16_t* hn = reinterpret_cast<uint16_t*>(sm);                 // H bf16
    float* lg = reinterpret_cast<float*>(sm + ((H * 2 + 15) & ~15)); // E fp32
    __shared__ float red[32];
    const int t = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int i = threadIdx.x * 8;

    if (hn_in) {
        *reinterpret_cast<uint4*>(hn + i) = *reinterpret_cast<const uint4*>(hn_in + static_cast<int64_t>(t) * H + i);
    } else {
        const float* xr = x + static_cast<int64_t>(t) * H + i;
        float v[8];
        {
            const float4 a = *reinterpret_cast<const float4*>(xr);
            const float4 b = *reinterpret_cast<const float4*>(xr + 4);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        }
        if (parts > 0) {
            // h = residual + sum of the O-projection split-K partials (fixed
            // order -> deterministic); h_out feeds the top-k combine
            float pv[4][8];  // partials 1..3 in registers (the runtime uses <= 4 splits)
#pragma unroll
            for (int p = 1; p < 4; ++p)
                if (p < parts) {
                    const float4 a = *reinterpret_cast<const float4*>(xr + p * part_stride);
                    const float4 b = *reinterpret_cast<const float4*>(xr + p * part_stride + 4);
                    pv[p][0] = a.x; pv[p][1] = a.y; pv[p][2] = a.z; pv[p][3] = a.w;
                    pv[p][4] = b.x; pv[p][5] = b.y; pv[p][6] = b.z; pv[p][7] = b.w;
                }
            const float* rr = residual + static_cast<int64_t>(t) * H + i;
            const float4 ra = *reinterpret_cast<const float4*>(rr);
            const float4 rb = *reinterpret_cast<const float4*>(rr + 4);
            const float rv[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
            for (int p = 1; p < 4; ++p)
                if (p < parts)
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] += pv[p][j];
            for (int p = 4; p < parts; ++p)  // further partials, same ascending order
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] += xr[p * part_stride + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += rv[j];
            float* hr = h_out + static_cast<int64_t>(t) * H + i;
            *reinterpret_cast<float4*>(hr) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4*>(hr + 4) = make_float4(v[4], v[5], v[6], v[7]);
        }
        float ss = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += v[j] * v[j];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
        if (lane == 0) red[warp] = ss;
        __syncthreads();
        float tot = 0.0f;
        for (int k = 0; k < nw; ++k) tot += red[k];
        const float r = 1.0f / sqrtf(tot / static_cast<float>(H) + eps);
        const uint4 gv = *reinterpret_cast<const uint4*>(gamma + i);
        const uint16_t* g = reinterpret_cast<const uint16_t*>(&gv);
        uint4 o;
        uint16_t* ob = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
        for (int j = 0; j < 8; ++j) ob[j] = f32_to_bf16_bits(v[j] * r * bf16_bits_to_f32(g[j]));
        *reinterpret_cast<uint4*>(hn + i) = o;
    }
    if (hn_out)
        *reinterpret_cast<uint4*>(hn_out + static_cast<int64_t>(t) * H + i) = *reinterpret_cast<const uint4*>(hn + i);
    __syncthreads();

    const int chunks = H / 8;
    for (int e = warp; e < E; e += nw) {
        const uint16_t* we = w + static_cast<int64_t>(e) * H;
        float acc = 0.0f;
        for (int c = lane; c < chunks; c += 32) {
            const uint4 xv = *reinterpret_cast<const uint4*>(hn + c * 8);
            const uint4 wv = *reinterpret_cast<const uint4*>(we + c * 8);
            const uint16_t* xb = reinterpret_cast<const uint16_t*>(&xv);
            const uint16_t* wb = reinterpret_cast<const uint16_t*>(&wv);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = __fmaf_rn(bf16_bits_to_f32(xb[j]), bf16_bits_to_f32(wb[j]), acc);
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, m));
        if (lane == 0) lg[e] = acc;
    }
    __syncthreads();
    if (logits)
        for (int e = threadIdx.x; e < E; e += blockDim.x) logits[static_cast<int64_t>(t) * E + e] = lg[e];
    if (threadIdx.x == 0) {
        // selection (ties -> lower index) and softmax over the k selected
        // logits; fully unrolled over k <= 8 so everything stays in registers
        uint64_t used = 0;
        float* sv = red;  // K <= 8 selected exp values (red is free again here)
        float top = 0.0f, sum = 0.0f;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            if (s < K) {
                int best = -1;
                float bv = 0.0f;
                for (int e = 0; e < E; ++e)
                    if (!((used >> e) & 1) && (best < 0 || lg[e] > bv)) {
                        best = e;
                        bv = lg[e];
                    }
                used |= 1ull << best;
                topk_idx[t * K + s] = best;
                if (s == 0) top = bv;
                sv[s] = expf(bv - top);
                sum += sv[s];
            }
        }
#pragma unroll
        for (int s = 0; s < 8; ++s)
            if (s < K) topk_w[t * K + s] = sv[s] / sum;
    }
}

__global__ void permute_kernel(const int32_t* topk_idx, const uint16_t* hn, int T, int H, int E,
                               int K, int32_t* counts, int32_t* offsets, int32_t* perm,
                               int32_t* inv, uint8_t* xp, int R) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    __shared__ int s_cnt[kMaxE];
    __shared__ int s_off[kMaxE + 1];
    extern __shared__ int dyn[];
    const int nt = blockDim.x, tid = threadIdx.x;
    int* hist = dyn;                    // [E][nt]: slots of expert e in thread t's run
    int* s_slot_row = dyn + E * nt;     // [T*K] padded row of each slot
    const int TK = T * K;
    // Slot i = t*K + s.  Thread t owns the contiguous run [t*per, (t+1)*per),
    // so "rank within expert = #earlier slots choosing e" is the exclusive
    // scan over threads of the per-run histograms plus the in-run count:
    // stable (expert, token, slot) order in one pass over the slots.
    const int per = (TK + nt - 1) / nt;
    const int i0 = min(TK, tid * per), i1 = min(TK, i0 + per);
    for (int e = 0; e < E; ++e) hist[e * nt + tid] = 0;
    for (int i = i0; i < i1; ++i) ++hist[topk_idx[i] * nt + tid];
    __syncthreads();
    {  // per expert: exclusive scan over the nt thread counts (one warp per expert)
        const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5, span = nt / 32;
        for (int e = warp; e < E; e += nw) {
            int* h = hist + e * nt + lane * span;
            int local = 0;
            for (int j = 0; j < span; ++j) local += h[j];
            int incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int run = incl - local;
            for (int j = 0; j < span; ++j) {
                const int c = h[j];
                h[j] = run;
                run += c;
            }
            if (lane == 31) s_cnt[e] = incl;
        }
    }
    __syncthreads();
    if (tid == 0) {
        s_off[0] = 0;
        for (int e = 0; e < E; ++e) s_off[e + 1] = s_off[e] + ((s_cnt[e] + 15) & ~15);
    }
    __syncthreads();
    for (int i = i0; i < i1; ++i) {
        const int e = topk_idx[i];
        s_slot_row[i] = s_off[e] + hist[e * nt + tid]++;
    }
    __syncthreads();
    const int rows = s_off[E];
    if (blockIdx.x == 0) {
        for (int e = threadIdx.x; e < E; e += blockDim.x) counts[e] = s_cnt[e];
        for (int e = threadIdx.x; e <= E; e += blockDim.x) offsets[e] = s_off[e];
        for (int r = threadIdx.x; r < R; r += blockDim.x) perm[r] = -1;
        __syncthreads();
        for (int i = threadIdx.x; i < TK; i += blockDim.x) {
            inv[i] = s_slot_row[i];
            perm[s_slot_row[i]] = i;
        }
    }
    // Gather: 16-byte chunks of (slot, k) distributed over the grid.
    const int cpr = H / 8;
    const int64_t work = static_cast<int64_t>(TK) * cpr;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < work;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(w / cpr), c = static_cast<int>(w % cpr);
        const int t = i / K;
        *reinterpret_cast<uint4*>(xp + b_packed_off(s_slot_row[i], c * 8, R)) =
            *reinterpret_cast<const uint4*>(hn + static_cast<int64_t>(t) * H + c * 8);
    }
    (void)rows;
}

}  // namespace

cudaError_t launch_router(const float* x, const uint16_t* gamma, float eps, const uint16_t* hn_in,
                          const uint16_t* w, int T, int H, int E, int K, uint16_t* hn_out,
                          float* logits, int32_t* topk_idx, float* topk_w, cudaStream_t s,
                          int parts, int64_t part_stride, const float* residual, float* h_out) {
    if (T <= 0) return cudaSuccess;
    if (H % 256 || E > kMaxE || K > 8 || K > E || (!hn_in && (!x || !gamma)) ||
        (parts > 0 && (!residual || !h_out)))
        return cudaErrorInvalidValue;
    if (H > 6144) return cudaErrorInvalidValue;  // H/8 threads per token
    const int smem = ((H * 2 + 15) & ~15) + E * 4;
    return launch_k(router_kernel, dim3(T), dim3(H / 8), smem, s, x, gamma, eps, hn_in, w, H, E, K, hn_out, logits, topk_idx,
                                       topk_w, parts, part_stride, residual, h_out);
}

cudaError_t launch_moe_permute(const int32_t* topk_idx, const uint16_t* hn, int T, int H, int E,
                               int K, int32_t* counts, int32_t* offsets, int32_t* perm,
                               int32_t* inv, uint8_t* xp, int R, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (E > kMaxE || T * K > kMaxSlots || H % 64 || R < T * K + 16 * E) return cudaErrorInvalidValue;
    const int64_t work = static_cast<int64_t>(T) * K * (H / 8);
    int grid = static_cast<int>((work + 255) / 256);
    if (grid > 296) grid = 296;
    if (grid < 1) grid = 1;
    const int smem = (E * 256 + T * K) * static_cast<int>(sizeof(int));
    if (const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(permute_kernel),
                                               (kMaxE * 256 + kMaxSlots) * static_cast<int>(sizeof(int)));
        e != cudaSuccess)
        return e;
    return launch_k(permute_kernel, dim3(grid), dim3(256), smem, s, topk_idx, hn, T, H, E, K, counts, offsets, perm, inv, xp, R);
}

}  // namespace mltk
