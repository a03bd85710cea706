// Bandwidth-bound glue kernels of the decode step: embedding gather,
// RMSNorm -> packed operand, row packing, RoPE (D1 layout), top-k combine
// and greedy argmax.  All vectorised 16-byte accesses; one CTA per token row
// (rows are 2-24 KiB at the shapes of BASELINE.json, so one CTA streams a
// row at full per-SM bandwidth and T >= 64 rows fill the chip).
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {

namespace {
bool g_pdl = false;
}
bool pdl_enabled() { return g_pdl; }
void set_pdl(bool on) { g_pdl = on; }

cudaError_t ensure_smem_attr(const void* kern, int bytes) {
    // the largest size set so far per (device, kernel); raised when a launch needs more
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find({dev, kern});
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); e != cudaSuccess)
        return e;
    done[{dev, kern}] = bytes;
    return cudaSuccess;
}

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
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
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

// Row kernels below use one CTA of H/8 threads per token: thread i owns the
// 8 consecutive elements [8i, 8i+8) of the row and issues all of its loads
// up front, so a CTA has the whole row (and every split-K partial) in
// flight at once instead of a latency-bound strided loop.
__device__ __forceinline__ float block_sum_rows(float v, float* red) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.0f;
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}

__device__ __forceinline__ void load_row8(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store_row8(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
// RMSNorm(v) * gamma of this thread's 8 elements -> one 16-byte bf16 chunk
__device__ __forceinline__ uint4 norm8(const float (&v)[8], float r, const uint16_t* gamma) {
    const uint4 gv = *reinterpret_cast<const uint4*>(gamma);
    const uint16_t* g = reinterpret_cast<const uint16_t*>(&gv);
    uint4 o;
    uint16_t* ob = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
    for (int j = 0; j < 8; ++j) ob[j] = f32_to_bf16_bits(v[j] * r * bf16_bits_to_f32(g[j]));
    return o;
}

__global__ void __launch_bounds__(1024) rmsnorm_pack_kernel(const float* x, const uint16_t* gamma, int H,
                                                            float eps, uint8_t* out, int R) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    __shared__ float red[32];
    const int t = blockIdx.x, i = threadIdx.x * 8;
    float v[8];
    load_row8(x + static_cast<int64_t>(t) * H + i, v);
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += v[j] * v[j];
    ss = block_sum_rows(ss, red);
    const float r = 1.0f / sqrtf(ss / static_cast<float>(H) + eps);
    *reinterpret_cast<uint4*>(out + b_packed_off(t, i, R)) = norm8(v, r, gamma + i);
}

__global__ void pack_rows_kernel(const uint16_t* src, int ld, int K, uint8_t* dst, int R) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    const int t = blockIdx.x;
    for (int i = threadIdx.x * 8; i < K; i += blockDim.x * 8)
        *reinterpret_cast<uint4*>(dst + b_packed_off(t, i, R)) =
            *reinterpret_cast<const uint4*>(src + static_cast<int64_t>(t) * ld + i);
}

// RoPE (rotate-half) over the q and k heads, copy of the v heads, fp32
// split-K partials summed on the fly (fixed order).  Work unit = 8
// consecutive rotation pairs of one q/k head (two 16-byte bf16 stores at i
// and i + d/2) or 8 dims of one v head; units are spread over the grid.
// With kv != nullptr (A_g = 1) the roped k and the v rows of this step are
// also stored into the swizzled paged pool at position pos[t] (the
// kv_append of the decode step fused into its producer).
template <int D>
__global__ void __launch_bounds__(256) rope_qkv_kernel(const float* __restrict__ qkv, int parts,
                                                       int64_t part_stride, const int32_t* __restrict__ pos,
                                                       const float2* __restrict__ rope, int T, int nq, int nkv,
                                                       uint16_t* __restrict__ out, KvAppend kv) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    constexpr int half = D / 2;
    constexpr int upr = half / 8;  // units per q/k head
    const int W = (nq + 2 * nkv) * D;
    const int units = (nq + nkv) * upr + nkv * (D / 8);
    const int64_t total = static_cast<int64_t>(T) * units;
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < total;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(u / units), j = static_cast<int>(u % units);
        const float* src = qkv + static_cast<int64_t>(t) * W;
        uint16_t* dst = out + static_cast<int64_t>(t) * W;
        auto load8 = [&](int col, float (&v)[8]) {
            float4 a = *reinterpret_cast<const float4*>(src + col);
            float4 b = *reinterpret_cast<const float4*>(src + col + 4);
            for (int p = 1; p < parts; ++p) {
                const float4 c = *reinterpret_cast<const float4*>(src + p * part_stride + col);
                const float4 e = *reinterpret_cast<const float4*>(src + p * part_stride + col + 4);
                a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
                b.x += e.x; b.y += e.y; b.z += e.z; b.w += e.w;
            }
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        };
        auto pack8 = [](const float (&v)[8]) {
            uint4 o;
            o.x = f32_to_bf16_bits(v[0]) | (static_cast<uint32_t>(f32_to_bf16_bits(v[1])) << 16);
            o.y = f32_to_bf16_bits(v[2]) | (static_cast<uint32_t>(f32_to_bf16_bits(v[3])) << 16);
            o.z = f32_to_bf16_bits(v[4]) | (static_cast<uint32_t>(f32_to_bf16_bits(v[5])) << 16);
            o.w = f32_to_bf16_bits(v[6]) | (static_cast<uint32_t>(f32_to_bf16_bits(v[7])) << 16);
            return o;
        };
        const int p_t = pos[t];
        uint16_t *kdst = nullptr, *vdst = nullptr;
        if (kv.k_pool) {
            const int id = kv.block_table[static_cast<int64_t>(kv.seq[t]) * kv.max_pages + p_t / kKvPage];
            kdst = kv.k_pool + static_cast<int64_t>(id) * nkv * kKvPage * D;
            vdst = kv.v_pool + static_cast<int64_t>(id) * nkv * kKvPage * D;
        }
        const int within = p_t % kKvPage;
        if (j < (nq + nkv) * upr) {
            const int head = j / upr, i0 = (j % upr) * 8;
            float a[8], b[8], ra[8], rb[8];
            load8(head * D + i0, a);
            load8(head * D + i0 + half, b);
            const float4* cs4 = reinterpret_cast<const float4*>(rope + static_cast<int64_t>(p_t) * half + i0);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float4 c = cs4[e];  // (cos, sin) of pairs i0+2e, i0+2e+1
                ra[2 * e] = a[2 * e] * c.x - b[2 * e] * c.y;
                rb[2 * e] = b[2 * e] * c.x + a[2 * e] * c.y;
                ra[2 * e + 1] = a[2 * e + 1] * c.z - b[2 * e + 1] * c.w;
                rb[2 * e + 1] = b[2 * e + 1] * c.z + a[2 * e + 1] * c.w;
            }
            const uint4 oa = pack8(ra), ob = pack8(rb);
            *reinterpret_cast<uint4*>(dst + head * D + i0) = oa;
            *reinterpret_cast<uint4*>(dst + head * D + i0 + half) = ob;
            if (kdst && head >= nq) {
                uint16_t* kh = kdst + static_cast<int64_t>(head - nq) * kKvPage * D;
                *reinterpret_cast<uint4*>(kh + kv_page_off(within, i0)) = oa;
                *reinterpret_cast<uint4*>(kh + kv_page_off(within, i0 + half)) = ob;
            }
        } else {
            const int jv = j - (nq + nkv) * upr;
            const int vh = jv / (D / 8), i0 = (jv % (D / 8)) * 8;
            float a[8];
            load8((nq + nkv + vh) * D + i0, a);
            const uint4 oa = pack8(a);
            *reinterpret_cast<uint4*>(dst + (nq + nkv + vh) * D + i0) = oa;
            if (vdst) *reinterpret_cast<uint4*>(vdst + static_cast<int64_t>(vh) * kKvPage * D + kv_page_off(within, i0)) = oa;
        }
    }
}

// x = h + sum_s w_s * y[inv[t,s]] (slot order); with gamma != nullptr the
// RMSNorm of the new x (the next layer's attention norm, or the final norm)
// is fused: packed bf16 row t of xn (capacity R) for the next projection.
template <int K>
__global__ void __launch_bounds__(768) combine_kernel(const float* h, const float* y, int ldy,
                                                      const int32_t* inv, const float* w, int H,
                                                      float* x, const uint16_t* gamma, float eps,
                                                      uint8_t* xn, int R, int n_parts, int64_t pstride) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    __shared__ float red[32];
    const int t = blockIdx.x, i = threadIdx.x * 8;
    float ys[K][8];  // every slot row's loads issued before the sum
#pragma unroll
    for (int s = 0; s < K; ++s) load_row8(y + static_cast<int64_t>(inv[t * K + s]) * ldy + i, ys[s]);
    // split-K partials of the down GEMM: summed in part order (deterministic)
    for (int p = 1; p < n_parts; ++p) {
#pragma unroll
        for (int s = 0; s < K; ++s) {
            float v[8];
            load_row8(y + p * pstride + static_cast<int64_t>(inv[t * K + s]) * ldy + i, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) ys[s][j] += v[j];
        }
    }
    float r[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (h) load_row8(h + static_cast<int64_t>(t) * H + i, r);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < K; ++s) {
        const float ws = w[t * K + s];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += ws * ys[s][j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = r[j] + acc[j];
    store_row8(x + static_cast<int64_t>(t) * H + i, acc);
    if (gamma) {
        float ss = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += acc[j] * acc[j];
        ss = block_sum_rows(ss, red);
        const float rr = 1.0f / sqrtf(ss / static_cast<float>(H) + eps);
        *reinterpret_cast<uint4*>(xn + b_packed_off(t, i, R)) = norm8(acc, rr, gamma + i);
    }
}

// out = sum_p parts[p*stride] (+ add): split-K reduction / residual add,
// fixed order (deterministic).
__global__ void sum_parts_kernel(const float* parts, int n_parts, int64_t stride, const float* add,
                                 float* out, int64_t n4) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
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
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
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
    return launch_k(embed_kernel, dim3(T), dim3(128), 0, s, tokens, table, H, x);
}

cudaError_t launch_rmsnorm_pack(const float* x, const uint16_t* gamma, int T, int H, float eps,
                                uint8_t* out, int R, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (H % 256 || H > 8192 || R < T) return cudaErrorInvalidValue;
    return launch_k(rmsnorm_pack_kernel, dim3(T), dim3(H / 8), 0, s, x, gamma, H, eps, out, R);
}

cudaError_t launch_pack_rows(const uint16_t* src, int ld, int T, int K, uint8_t* dst, int R,
                             cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (K % 64 || R < T) return cudaErrorInvalidValue;
    return launch_k(pack_rows_kernel, dim3(T), dim3(128), 0, s, src, ld, K, dst, R);
}

cudaError_t launch_rope_qkv(const float* qkv, int parts, int64_t part_stride, const int32_t* pos,
                            const float2* rope, int T, int nq, int nkv, int d, uint16_t* out,
                            cudaStream_t s, const KvAppend* kv) {
    if (T <= 0) return cudaSuccess;
    if (parts < 1 || d != 128 || part_stride % 4) return cudaErrorInvalidValue;
    const int64_t total = static_cast<int64_t>(T) * ((nq + nkv) * 8 + nkv * 16);
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    return launch_k(rope_qkv_kernel<128>, dim3(grid), dim3(256), 0, s, qkv, parts, part_stride, pos, rope, T, nq, nkv, out,
                                              kv ? *kv : KvAppend{});
}

cudaError_t launch_moe_combine(const float* h, const float* y, int ldy, const int32_t* inv,
                               const float* w, int T, int H, int K, float* x, cudaStream_t s,
                               const uint16_t* gamma, float eps, uint8_t* xn, int R, int n_parts,
                               int64_t part_stride) {
    if (T <= 0) return cudaSuccess;
    if (H % 256 || H > 6144 || ldy % 4 || (gamma && (!xn || R < T)) || n_parts < 1 || part_stride % 4)
        return cudaErrorInvalidValue;
    switch (K) {  // x = h + sum of K slot rows (slot order)
        case 1: return launch_k(combine_kernel<1>, dim3(T), dim3(H / 8), 0, s, h, y, ldy, inv, w, H, x, gamma, eps, xn, R, n_parts, part_stride);
        case 2: return launch_k(combine_kernel<2>, dim3(T), dim3(H / 8), 0, s, h, y, ldy, inv, w, H, x, gamma, eps, xn, R, n_parts, part_stride);
        case 4: return launch_k(combine_kernel<4>, dim3(T), dim3(H / 8), 0, s, h, y, ldy, inv, w, H, x, gamma, eps, xn, R, n_parts, part_stride);
        case 8: return launch_k(combine_kernel<8>, dim3(T), dim3(H / 8), 0, s, h, y, ldy, inv, w, H, x, gamma, eps, xn, R, n_parts, part_stride);
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_sum_parts(const float* parts, int n_parts, int64_t stride, const float* add,
                             float* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (n % 4 || stride % 4 || n_parts < 1) return cudaErrorInvalidValue;
    const int64_t n4 = n / 4;
    int grid = static_cast<int>((n4 + 255) / 256);
    if (grid > 1184) grid = 1184;
    return launch_k(sum_parts_kernel, dim3(grid), dim3(256), 0, s, parts, n_parts, stride, add, out, n4);
}

cudaError_t launch_argmax(const float* logits, int T, int V, int32_t* ids, float* margin,
                          cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    return launch_k(argmax_kernel, dim3(T), dim3(512), 0, s, logits, V, ids, margin);
}

}  // namespace mltk
