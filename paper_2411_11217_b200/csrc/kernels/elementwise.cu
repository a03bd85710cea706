// Bandwidth-bound glue kernels of the decode step: embedding gather,
// RMSNorm -> packed operand, row packing, RoPE (D1 layout), top-k combine
// and greedy argmax.  All vectorised 16-byte accesses; one CTA per token row
// (rows are 2-24 KiB at the shapes of BASELINE.json, so one CTA streams a
// row at full per-SM bandwidth and T >= 64 rows fill the chip).
#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.0f;
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}

__global__ void embed_kernel(const int32_t* tokens, const uint16_t* table, int H, float* x) {
    const int t = blockIdx.x;
    const uint16_t* src = table + static_cast<int64_t>(tokens[t]) * H;
    for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + i);
        const uint16_t* e = reinterpret_cast<const uint16_t*>(&v);
        float4 a, b;
        a.x = bf16_bits_to_f32(e[0]); a.y = bf16_bits_to_f32(e[1]);
        a.z = bf16_bits_to_f32(e[2]); a.w = bf16_bits_to_f32(e[3]);
        b.x = bf16_bits_to_f32(e[4]); b.y = bf16_bits_to_f32(e[5]);
        b.z = bf16_bits_to_f32(e[6]); b.w = bf16_bits_to_f32(e[7]);
        float4* d = reinterpret_cast<float4*>(x + static_cast<int64_t>(t) * H + i);
        d[0] = a;
        d[1] = b;
    }
}

__global__ void rmsnorm_pack_kernel(const float* x, const uint16_t* gamma, int H, float eps,
                                    uint8_t* out, int R) {
    __shared__ float red[32];
    const int t = blockIdx.x;
    const float* xr = x + static_cast<int64_t>(t) * H;
    float ss = 0.0f;
    for (int i = threadIdx.x * 4; i < H; i += blockDim.x * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xr + i);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = block_sum(ss, red);
    const float r = 1.0f / sqrtf(ss / static_cast<float>(H) + eps);
    for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
        const float4 a = *reinterpret_cast<const float4*>(xr + i);
        const float4 b = *reinterpret_cast<const float4*>(xr + i + 4);
        const uint4 gv = *reinterpret_cast<const uint4*>(gamma + i);
        const uint16_t* g = reinterpret_cast<const uint16_t*>(&gv);
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint4 o;
        uint16_t* ob = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
        for (int j = 0; j < 8; ++j) ob[j] = f32_to_bf16_bits(v[j] * r * bf16_bits_to_f32(g[j]));
        *reinterpret_cast<uint4*>(out + b_packed_off(t, i, R)) = o;
    }
}

__global__ void pack_rows_kernel(const uint16_t* src, int ld, int K, uint8_t* dst, int R) {
    const int t = blockIdx.x;
    for (int i = threadIdx.x * 8; i < K; i += blockDim.x * 8)
        *reinterpret_cast<uint4*>(dst + b_packed_off(t, i, R)) =
            *reinterpret_cast<const uint4*>(src + static_cast<int64_t>(t) * ld + i);
}

// One CTA per token; thread j < (nq+nkv)*half handles one rotation pair, the
// v part is copied.
// Sums the split-K partials of the QKV projection (parts >= 1) on the fly.
__global__ void rope_qkv_kernel(const float* qkv, int parts, int64_t part_stride, const int32_t* pos,
                                const float2* rope, int nq, int nkv, int d, uint16_t* out) {
    const int t = blockIdx.x;
    const int half = d / 2;
    const int W = (nq + 2 * nkv) * d;
    const float* src = qkv + static_cast<int64_t>(t) * W;
    uint16_t* dst = out + static_cast<int64_t>(t) * W;
    const float2* cs = rope + static_cast<int64_t>(pos[t]) * half;
    auto at = [&](int j) {
        float v = src[j];
        for (int p = 1; p < parts; ++p) v += src[p * part_stride + j];
        return v;
    };
    const int pairs = (nq + nkv) * half;
    for (int j = threadIdx.x; j < pairs; j += blockDim.x) {
        const int head = j / half, i = j % half;
        const float c = cs[i].x, s = cs[i].y;
        const float a = at(head * d + i), b = at(head * d + i + half);
        dst[head * d + i] = f32_to_bf16_bits(a * c - b * s);
        dst[head * d + i + half] = f32_to_bf16_bits(b * c + a * s);
    }
    for (int j = (nq + nkv) * d + threadIdx.x; j < W; j += blockDim.x)
        dst[j] = f32_to_bf16_bits(at(j));
}

__global__ void combine_kernel(const float* h, const float* y, int ldy, const int32_t* inv,
                               const float* w, int H, int K, float* x) {
    const int t = blockIdx.x;
    for (int i = threadIdx.x * 4; i < H; i += blockDim.x * 4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < K; ++s) {
            const float ws = w[t * K + s];
            const float4 v = *reinterpret_cast<const float4*>(y + static_cast<int64_t>(inv[t * K + s]) * ldy + i);
            acc.x += ws * v.x; acc.y += ws * v.y; acc.z += ws * v.z; acc.w += ws * v.w;
        }
        const float4 r = h ? *reinterpret_cast<const float4*>(h + static_cast<int64_t>(t) * H + i)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(x + static_cast<int64_t>(t) * H + i) =
            make_float4(r.x + acc.x, r.y + acc.y, r.z + acc.z, r.w + acc.w);
    }
}

// out = sum_p parts[p*stride] (+ add): split-K reduction / residual add,
// fixed order (deterministic).
__global__ void sum_parts_kernel(const float* parts, int n_parts, int64_t stride, const float* add,
                                 float* out, int64_t n4) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 a = reinterpret_cast<const float4*>(parts)[i];
        for (int p = 1; p < n_parts; ++p) {
            const float4 b = reinterpret_cast<const float4*>(parts + p * stride)[i];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        if (add) {
            const float4 b = reinterpret_cast<const float4*>(add)[i];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        reinterpret_cast<float4*>(out)[i] = a;
    }
}

struct Best2 {
    float v1;
    int i1;
    float v2;
};

__device__ __forceinline__ bool better(float a, int ia, float b, int ib) {
    return a > b || (a == b && ia < ib);
}

__device__ __forceinline__ void merge(Best2& a, const Best2& b) {
    if (better(b.v1, b.i1, a.v1, a.i1)) {
        a.v2 = fmaxf(a.v1, b.v2);
        a.v1 = b.v1;
        a.i1 = b.i1;
    } else {
        a.v2 = fmaxf(a.v2, b.v1);
    }
}

__global__ void argmax_kernel(const float* logits, int V, int32_t* ids, float* margin) {
    __shared__ Best2 red[32];
    const int t = blockIdx.x;
    const float* r = logits + static_cast<int64_t>(t) * V;
    Best2 b{-FLT_MAX, 0x7fffffff, -FLT_MAX};
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const Best2 c{r[i], i, -FLT_MAX};
        merge(b, c);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        Best2 o;
        o.v1 = __shfl_xor_sync(0xffffffffu, b.v1, m);
        o.i1 = __shfl_xor_sync(0xffffffffu, b.i1, m);
        o.v2 = __shfl_xor_sync(0xffffffffu, b.v2, m);
        merge(b, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best2 f = red[0];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) merge(f, red[k]);
        ids[t] = f.i1;
        if (margin) margin[t] = f.v1 - f.v2;
    }
}

}  // namespace

cudaError_t launch_embed(const int32_t* tokens, const uint16_t* table, int T, int H, float* x,
                         cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (H % 8) return cudaErrorInvalidValue;
    embed_kernel<<<T, 128, 0, s>>>(tokens, table, H, x);
    return cudaGetLastError();
}

cudaError_t launch_rmsnorm_pack(const float* x, const uint16_t* gamma, int T, int H, float eps,
                                uint8_t* out, int R, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (H % 64 || R < T) return cudaErrorInvalidValue;
    rmsnorm_pack_kernel<<<T, 256, 0, s>>>(x, gamma, H, eps, out, R);
    return cudaGetLastError();
}

cudaError_t launch_pack_rows(const uint16_t* src, int ld, int T, int K, uint8_t* dst, int R,
                             cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (K % 64 || R < T) return cudaErrorInvalidValue;
    pack_rows_kernel<<<T, 128, 0, s>>>(src, ld, K, dst, R);
    return cudaGetLastError();
}

cudaError_t launch_rope_qkv(const float* qkv, int parts, int64_t part_stride, const int32_t* pos,
                            const float2* rope, int T, int nq, int nkv, int d, uint16_t* out,
                            cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (parts < 1) return cudaErrorInvalidValue;
    rope_qkv_kernel<<<T, 256, 0, s>>>(qkv, parts, part_stride, pos, rope, nq, nkv, d, out);
    return cudaGetLastError();
}

cudaError_t launch_moe_combine(const float* h, const float* y, int ldy, const int32_t* inv,
                               const float* w, int T, int H, int K, float* x, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (H % 4 || ldy % 4) return cudaErrorInvalidValue;
    combine_kernel<<<T, 256, 0, s>>>(h, y, ldy, inv, w, H, K, x);
    return cudaGetLastError();
}

cudaError_t launch_sum_parts(const float* parts, int n_parts, int64_t stride, const float* add,
                             float* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (n % 4 || stride % 4 || n_parts < 1) return cudaErrorInvalidValue;
    const int64_t n4 = n / 4;
    int grid = static_cast<int>((n4 + 255) / 256);
    if (grid > 1184) grid = 1184;
    sum_parts_kernel<<<grid, 256, 0, s>>>(parts, n_parts, stride, add, out, n4);
    return cudaGetLastError();
}

cudaError_t launch_argmax(const float* logits, int T, int V, int32_t* ids, float* margin,
                          cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    argmax_kernel<<<T, 512, 0, s>>>(logits, V, ids, margin);
    return cudaGetLastError();
}

}  // namespace mltk
