// Causal GQA attention for the prefill stage (PAPER.md:166 — "the prompt
// tokens' keys and values are computed and stored"; the prefill runs
// entirely on the GPU).
//
// Inputs are the roped bf16 rows the QKV stage writes for a chunk of prompt
// tokens, [T][W] with W = (n_q + 2 n_kv) d; sequences are contiguous row
// ranges and never split across chunks, so every key a query needs is in the
// same buffer.  Output is the packed bf16 B operand of the O projection.
//
// One CTA per (16-query tile of one sequence, kv head); warp w handles query
// head kvh*G + w for the 16 queries, so all G heads of a group share the K/V
// tiles in shared memory (GQA reuse).  Key tiles of 64 are double-buffered
// with cp.async into an XOR-swizzled layout (16-byte chunk c of row r at
// c ^ (r & 7)) that makes every ldmatrix phase conflict-free.  S = Q K^T and
// O += P V run on mma.sync m16n8k16 bf16 -> fp32; softmax is online in the
// exp2 domain.  Prefill attention is ~3% of a Mixtral prefill layer's FLOPs
// (planner.cpp:112-124), so this kernel uses the warp-level MMA rather than
// tcgen05.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kD = 128;         // head dim (runtime requires 128)
constexpr int kQ = 16;          // queries per CTA
constexpr int kKT = 64;         // keys per tile
constexpr int kRowBytes = kD * 2;
constexpr int kTileBytes = kKT * kRowBytes;  // 16 KiB

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
    return static_cast<uint32_t>(row * kRowBytes + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int n = valid ? 16 : 0;  // zero-fill rows past the sequence end
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

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

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return static_cast<uint32_t>(f32_to_bf16_bits(lo)) | (static_cast<uint32_t>(f32_to_bf16_bits(hi)) << 16);
}

// tiles[i] = {first row of the sequence in the chunk, sequence length, first query position}
__global__ void __launch_bounds__(256) prefill_attn_kernel(const uint16_t* __restrict__ qkv, int W,
                                                           const int4* __restrict__ tiles, int nq, int nkv,
                                                           float scale_log2, uint8_t* __restrict__ out, int R) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    extern __shared__ __align__(128) uint8_t smem[];
    const int4 tile = tiles[blockIdx.x];
    const int row0 = tile.x, len = tile.y, q0 = tile.z;
    const int kvh = blockIdx.y;
    const int G = nq / nkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int hq = kvh * G + warp;
    const int nthreads = blockDim.x;

    const int kend = min(len, q0 + kQ);  // keys [0, kend) are visible to some query of the tile
    const int ntiles = (kend + kKT - 1) / kKT;
    const uint16_t* kbase = qkv + static_cast<int64_t>(row0) * W + (nq + kvh) * kD;
    const uint16_t* vbase = qkv + static_cast<int64_t>(row0) * W + (nq + nkv + kvh) * kD;
    const uint32_t sk0 = smem_u32(smem), sv0 = sk0 + 2 * kTileBytes;

    auto load_tile = [&](int t, int buf) {
        const int kt0 = t * kKT;
        for (int i = threadIdx.x; i < kKT * 16; i += nthreads) {
            const int r = i >> 4, c = i & 15;
            const bool ok = kt0 + r < kend;
            const int64_t off = static_cast<int64_t>(ok ? kt0 + r : 0) * W + c * 8;
            cp_async16(sk0 + buf * kTileBytes + swz(r, c), kbase + off, ok);
            cp_async16(sv0 + buf * kTileBytes + swz(r, c), vbase + off, ok);
        }
        cp_async_commit();
    };
    load_tile(0, 0);

    // Q fragments (A operand, 16 x 128): rows g / g+8, cols 16kk + 2tig (+8)
    uint32_t qa[8][4];
    {
        const int qa_row = min(q0 + g, len - 1), qb_row = min(q0 + g + 8, len - 1);
        const uint16_t* qr0 = qkv + static_cast<int64_t>(row0 + qa_row) * W + hq * kD;
        const uint16_t* qr1 = qkv + static_cast<int64_t>(row0 + qb_row) * W + hq * kD;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qa[kk][0] = *reinterpret_cast<const uint32_t*>(qr0 + kk * 16 + 2 * tig);
            qa[kk][1] = *reinterpret_cast<const uint32_t*>(qr1 + kk * 16 + 2 * tig);
            qa[kk][2] = *reinterpret_cast<const uint32_t*>(qr0 + kk * 16 + 8 + 2 * tig);
            qa[kk][3] = *reinterpret_cast<const uint32_t*>(qr1 + kk * 16 + 8 + 2 * tig);
        }
    }

    float o[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const int qp0 = q0 + g, qp1 = q0 + g + 8;  // query positions of this thread's two rows

    for (int t = 0; t < ntiles; ++t) {
        const int buf = t & 1;
        if (t + 1 < ntiles) {
            load_tile(t + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const uint32_t sk = sk0 + buf * kTileBytes, sv = sv0 + buf * kTileBytes;
        const int kt0 = t * kKT;

        // S = Q K^T (16 x 64): 8 n-tiles of 8 keys
        float s[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
            for (int np = 0; np < 4; ++np) {  // n-tile pair (16 keys)
                const int mi = lane >> 3;
                const int row = np * 16 + (mi >> 1) * 8 + (lane & 7);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sk + swz(row, 2 * kk + (mi & 1)), b0, b1, b2, b3);
                mma16816(s[2 * np], qa[kk], b0, b1);
                mma16816(s[2 * np + 1], qa[kk], b2, b3);
            }
        }
        // causal / length mask and online softmax (exp2 domain)
        const bool need_mask = kt0 + kKT > q0;  // tile reaches the diagonal or the end
        float mx0 = m0, mx1 = m1;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int kp = kt0 + j * 8 + 2 * tig + e;
                float v0 = s[j][e] * scale_log2, v1 = s[j][2 + e] * scale_log2;
                if (need_mask) {
                    if (kp > qp0 || kp >= len) v0 = -INFINITY;
                    if (kp > qp1 || kp >= len) v1 = -INFINITY;
                }
                s[j][e] = v0;
                s[j][2 + e] = v1;
                mx0 = fmaxf(mx0, v0);
                mx1 = fmaxf(mx1, v1);
            }
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        // rows with no visible key yet keep m = -inf; use 0 as the exp base then
        const float b0 = mx0 == -INFINITY ? 0.f : mx0, b1 = mx1 == -INFINITY ? 0.f : mx1;
        const float c0 = exp2f(m0 - b0), c1 = exp2f(m1 - b1);  // m = -inf -> 0
        m0 = mx0;
        m1 = mx1;
        float rs0 = 0.f, rs1 = 0.f;
        uint32_t pa[4][4];  // P as A fragments: k-step j covers keys 16j..16j+15
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float p00 = exp2f(s[j][0] - b0), p01 = exp2f(s[j][1] - b0);
            const float p10 = exp2f(s[j][2] - b1), p11 = exp2f(s[j][3] - b1);
            rs0 += p00 + p01;
            rs1 += p10 + p11;
            pa[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p00, p01);
            pa[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p10, p11);
        }
        l0 = l0 * c0 + rs0;
        l1 = l1 * c1 + rs1;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            o[j][0] *= c0;
            o[j][1] *= c0;
            o[j][2] *= c1;
            o[j][3] *= c1;
        }
        // O += P V (16 x 128): k-steps of 16 keys, d-tile pairs of 16
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
            for (int dp = 0; dp < 8; ++dp) {
                const int mi = lane >> 3;
                const int row = ks * 16 + (mi & 1) * 8 + (lane & 7);
                uint32_t v0, v1, v2, v3;
                ldsm_x4_t(sv + swz(row, 2 * dp + (mi >> 1)), v0, v1, v2, v3);
                mma16816(o[2 * dp], pa[ks], v0, v1);
                mma16816(o[2 * dp + 1], pa[ks], v2, v3);
            }
        }
        __syncthreads();  // buffer buf is refilled by the next iteration's prefetch
    }

    // finalize: row sums across the quad, normalise, packed bf16 out
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int col = hq * kD + j * 8 + 2 * tig;
        if (qp0 < len)
            *reinterpret_cast<uint32_t*>(out + b_packed_off(row0 + qp0, col, R)) = pack_bf16(o[j][0] * i0, o[j][1] * i0);
        if (qp1 < len)
            *reinterpret_cast<uint32_t*>(out + b_packed_off(row0 + qp1, col, R)) = pack_bf16(o[j][2] * i1, o[j][3] * i1);
    }
}

// Rows of each sequence's roped K and V into a staging buffer laid out per
// sequence as [n_kv][len][d], so one strided copy per sequence lands them in
// the head-major host KV cache ([layer][seq][n_kv][max_ctx][d]).
__global__ void kv_stage_kernel(const uint16_t* __restrict__ qkv, int W, int nq, int nkv,
                                const int32_t* __restrict__ tok_seq, const int32_t* __restrict__ tok_pos,
                                const int32_t* __restrict__ seq_row0, const int32_t* __restrict__ seq_len,
                                int T, uint16_t* __restrict__ sk, uint16_t* __restrict__ sv) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    const int chunks = nkv * kD / 8;  // 16-byte chunks per token for K (same for V)
    const int64_t work = static_cast<int64_t>(T) * chunks;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < work;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(w / chunks), c = static_cast<int>(w % chunks);
        const int h = c / (kD / 8), i8 = c % (kD / 8);
        const int s = tok_seq[r], p = tok_pos[r];
        const int64_t dst = (static_cast<int64_t>(seq_row0[s]) * nkv + static_cast<int64_t>(h) * seq_len[s] + p) * kD + i8 * 8;
        const uint16_t* src = qkv + static_cast<int64_t>(r) * W;
        *reinterpret_cast<uint4*>(sk + dst) = *reinterpret_cast<const uint4*>(src + (nq + h) * kD + i8 * 8);
        *reinterpret_cast<uint4*>(sv + dst) = *reinterpret_cast<const uint4*>(src + (nq + nkv + h) * kD + i8 * 8);
    }
}

// x rows idx[i] -> dst row i (fp32), for the last-token lm_head of a chunk.
__global__ void gather_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ idx, int n, int H,
                                   float* __restrict__ dst) {
    pdl_trigger();  // dependents may launch; our inputs: after the wait
    pdl_wait();
    const int i = blockIdx.x;
    if (i >= n) return;
    const float4* s = reinterpret_cast<const float4*>(x + static_cast<int64_t>(idx[i]) * H);
    float4* d = reinterpret_cast<float4*>(dst + static_cast<int64_t>(i) * H);
    for (int c = threadIdx.x; c < H / 4; c += blockDim.x) d[c] = s[c];
}

}  // namespace

int prefill_attention_smem_bytes() { return 4 * kTileBytes; }

cudaError_t launch_prefill_attention(const uint16_t* qkv, int W, const int4* tiles, int n_tiles, int nq, int nkv,
                                     int d, uint8_t* out, int R, cudaStream_t s) {
    if (n_tiles <= 0) return cudaSuccess;
    if (d != kD || nkv <= 0 || nq % nkv || nq / nkv > 8 || W != (nq + 2 * nkv) * kD || R % 16)
        return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(prefill_attn_kernel),
                                         prefill_attention_smem_bytes());
        e != cudaSuccess)
        return e;
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(kD));
    return launch_k(prefill_attn_kernel, dim3(n_tiles, nkv), dim3(32 * (nq / nkv)), prefill_attention_smem_bytes(), s,
        qkv, W, tiles, nq, nkv, scale_log2, out, R);
}

cudaError_t launch_kv_stage(const uint16_t* qkv, int W, int nq, int nkv, int d, const int32_t* tok_seq,
                            const int32_t* tok_pos, const int32_t* seq_row0, const int32_t* seq_len, int T,
                            uint16_t* stage_k, uint16_t* stage_v, cudaStream_t s) {
    if (T <= 0) return cudaSuccess;
    if (d != kD) return cudaErrorInvalidValue;
    const int64_t work = static_cast<int64_t>(T) * nkv * kD / 8;
    int grid = static_cast<int>((work + 255) / 256);
    if (grid > 148 * 8) grid = 148 * 8;
    return launch_k(kv_stage_kernel, dim3(grid), dim3(256), 0, s, qkv, W, nq, nkv, tok_seq, tok_pos, seq_row0, seq_len, T, stage_k, stage_v);
}

cudaError_t launch_gather_rows(const float* x, const int32_t* idx, int n, int H, float* dst, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (H % 4) return cudaErrorInvalidValue;
    return launch_k(gather_rows_kernel, dim3(n), dim3(256), 0, s, x, idx, n, H, dst);
}

}  // namespace mltk
