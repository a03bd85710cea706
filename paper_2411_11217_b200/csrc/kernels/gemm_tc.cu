// Weight-streaming grouped GEMM on tcgen05 / TMEM, fed by 1-D bulk copies
// from the paged weight pool.  One kernel serves every projection of the
// decode step:
//   * dense linears (QKV, O + residual, lm_head): G = 1, one matrix;
//   * expert gate/up (SURVEY.md §2c `expert_gateup_silu`): G = n_e experts,
//     two matrices (W1, W3) sharing the token operand, SiLU(g)*u fused in
//     the TMEM epilogue, written straight into the packed operand layout of
//     the down projection;
//   * expert down (`expert_down`): G = n_e, one matrix, fp32 rows per
//     (expert, token) slot for the deterministic top-k combine.
//
// Swap-AB: the weight rows fill UMMA M = 128, the (few) tokens of a group
// fill N in {16..256}; D^T = W X^T accumulates in TMEM (128 lanes x N fp32
// columns per matrix).  The kernel is HBM-bound at decode sizes (intensity
// mu*k/n_e << ridge), so the design goal is to keep every SM's copy queue
// full: warp 0 streams 16 KiB weight tiles (L2 evict_first) + the token tile
// (evict_last) into a multi-stage smem ring, warp 1 issues the MMAs from one
// elected lane and commits stages back, warps 2-5 drain TMEM.  Weight tiles
// are addressed through a page table (one pointer per row block), which is
// how the same kernel reads resident rows and rows paged into either pool
// slot (runtime/weights.cpp).
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kThreads = 192;  // warp0 producer, warp1 MMA, warps2-5 epilogue
constexpr int kMaxMats = 2;
constexpr int kCtlBytes = 256;           // barriers + TMEM base
constexpr int kEpiScratch = 4 * 2048;    // per epilogue warp: 16 x 32 fp32 transpose tile

struct Smem {
    uint64_t full[8];
    uint64_t empty[8];
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint32_t tmem_base;
};

static_assert(sizeof(Smem) <= kCtlBytes, "control block fits its reserved bytes");

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const GemmArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KiB alignment for the SWIZZLE_128B atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    const int a_bytes = a.n_mats * kATileBytes;
    const int b_bytes = a.n_cap * 128;
    const int stage_bytes = a_bytes + b_bytes;
    const int stages = a.stages;
    Smem* ctl = reinterpret_cast<Smem*>(smem + stages * stage_bytes);

    const uint32_t warp = warp_idx_sync();
    const uint32_t lane = threadIdx.x & 31;
    if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[0], globaltimer());
    unsigned long long* const tr = a.trace ? a.trace + blockIdx.x * 8 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = globaltimer();
    const int acc_cols = a.n_mats * a.n_cap;     // TMEM columns per accumulator stage
    const int acc_stages = a.acc_stages;          // 1 or 2

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&ctl->full[s], 1);
            mbar_init(&ctl->empty[s], 1);
        }
        for (int s = 0; s < acc_stages; ++s) {
            mbar_init(&ctl->tfull[s], 1);
            mbar_init(&ctl->tempty[s], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&ctl->tmem_base, a.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = ctl->tmem_base;
    if (tr && threadIdx.x == 0) tr[1] = globaltimer();

    // virtual tile = (row block, group, N-chunk, K-split), K-split fastest
    const int n_virtual = a.G * a.RB * a.n_chunks * a.k_splits;
    const int KB = a.K / kBlockK;

    if (warp == 0) {
        // ===== producer =====
        if (elect_one()) {
            const uint64_t pol_w = l2_evict_first(), pol_x = l2_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
                const int ks = v % a.k_splits, u = v / a.k_splits;
                const int c = u % a.n_chunks, g = (u / a.n_chunks) % a.G, rb = u / a.n_chunks / a.G;
                const int kb0 = ks * KB / a.k_splits, kb1 = (ks + 1) * KB / a.k_splits;
                const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
                if (rows <= 0) continue;
                const int row0 = a.b_off ? a.b_off[g] : 0;
                const uint8_t* ab[kMaxMats];
                for (int mt = 0; mt < a.n_mats; ++mt)
                    ab[mt] = a.a_table[(static_cast<int64_t>(mt) * a.G + g) * a.RB + rb];
                for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                    const int nt = min(a.n_cap, rows - n0);
                    const int ntp = (nt + 15) & ~15;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&ctl->empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * stage_bytes;
                        uint8_t* sb = sa + a_bytes;
                        if (tr && v == static_cast<int>(blockIdx.x) && kb == kb0 && n0 == c * a.n_cap)
                            tr[2] = globaltimer();
                        mbar_expect_tx(&ctl->full[stage], a.n_mats * kATileBytes + ntp * 128);
                        for (int mt = 0; mt < a.n_mats; ++mt)
                            bulk_g2s(sa + mt * kATileBytes, ab[mt] + static_cast<int64_t>(kb) * kATileBytes,
                                     kATileBytes, &ctl->full[stage], pol_w);
                        const uint8_t* src = a.b + static_cast<int64_t>(kb) * a.R * 128 +
                                             static_cast<int64_t>(row0 + n0) * 128;
                        bulk_g2s(sb, src, ntp * 128, &ctl->full[stage], pol_x);
                        if (++stage == stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
            const int ks = v % a.k_splits, u = v / a.k_splits;
            const int c = u % a.n_chunks, g = (u / a.n_chunks) % a.G;
            const int kb0 = ks * KB / a.k_splits, kb1 = (ks + 1) * KB / a.k_splits;
            const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
            if (rows <= 0) continue;
            for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                const int nt = min(a.n_cap, rows - n0);
                const int ntp = (nt + 15) & ~15;
                const uint32_t idesc = idesc_bf16(128, ntp);
                mbar_wait(&ctl->tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d0 = tmem + acc * acc_cols;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&ctl->full[stage], phase);
                    tc_fence_after();
                    if (tr && lane == 0 && v == static_cast<int>(blockIdx.x) && kb == kb0 && n0 == c * a.n_cap)
                        tr[3] = globaltimer();
                    if (elect_one()) {
                        const uint32_t sa = smem_u32(smem + stage * stage_bytes);
                        const uint32_t sb = sa + a_bytes;
#pragma unroll
                        for (int k = 0; k < kBlockK / 16; ++k) {
                            const uint64_t bd = sdesc_sw128(sb + k * 32);
                            for (int mt = 0; mt < a.n_mats; ++mt)
                                umma_bf16(d0 + mt * a.n_cap, sdesc_sw128(sa + mt * kATileBytes + k * 32),
                                          bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                        }
                        umma_commit(&ctl->empty[stage]);
                        if (kb == kb1 - 1) umma_commit(&ctl->tfull[acc]);
                    }
                    __syncwarp();
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
                if (++acc == acc_stages) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> global =====
        const uint32_t quarter = warp & 3;  // TMEM lanes this warp may access
        float* const scr = reinterpret_cast<float*>(smem + stages * stage_bytes + kCtlBytes) + quarter * 512;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
            const int ks = v % a.k_splits, u = v / a.k_splits;
            const int c = u % a.n_chunks, g = (u / a.n_chunks) % a.G, rb = u / a.n_chunks / a.G;
            const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
            if (rows <= 0) continue;
            const int row0 = a.b_off ? a.b_off[g] : 0;
            const int mbase = rb * kBlockM + quarter * 32;  // this warp's 32 output features
            // K-split partials go to separate buffers, reduced by the consumer
            float* const outp = a.out_f32 ? a.out_f32 + static_cast<int64_t>(ks) * a.split_stride : nullptr;
            const float* const resid = a.k_splits == 1 ? a.residual : nullptr;
            for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                const int nt = min(a.n_cap, rows - n0);
                mbar_wait(&ctl->tfull[acc], acc_phase);
                tc_fence_after();
                if (tr && warp == 2 && lane == 0 && v == static_cast<int>(blockIdx.x) && n0 == c * a.n_cap)
                    tr[5] = globaltimer();
                const uint32_t t0 = tmem + ((quarter * 32u) << 16) + acc * acc_cols;
                // Each 32-feature x 16-token chunk goes TMEM -> registers ->
                // a per-warp smem transpose -> 16-byte global stores along the
                // feature axis (row-contiguous in the output), instead of 16
                // scalar stores per thread (6x slower, tools/trace_gemm.py).
                for (int c2 = 0; c2 < nt; c2 += 32) {
                    // issue the TMEM loads of two 16-token chunks (both matrices
                    // for SiLU), then a single wait: one TMEM round trip per 32 tokens
                    const bool two = c2 + 16 < nt;
                    uint32_t r0[2][16], r1[2][16];
                    tmem_ld16_async(t0 + c2, r0[0]);
                    if (two) tmem_ld16_async(t0 + c2 + 16, r0[1]);
                    if (a.epi != kEpiF32) {
                        tmem_ld16_async(t0 + a.n_cap + c2, r1[0]);
                        if (two) tmem_ld16_async(t0 + a.n_cap + c2 + 16, r1[1]);
                    }
                    tmem_wait_ld();
                    tmem_regs_ready(r0[0]);
                    if (two) tmem_regs_ready(r0[1]);
                    if (a.epi != kEpiF32) {
                        tmem_regs_ready(r1[0]);
                        if (two) tmem_regs_ready(r1[1]);
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = c2 + 16 * h;
                        if (c >= nt) break;
                        if (a.epi == kEpiF32) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) scr[j * 32 + lane] = __uint_as_float(r0[h][j]) * a.alpha;
                            __syncwarp();
                            const int f = (lane & 7) * 4;
                            float4 rv[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {  // residual loads first (all in flight)
                                const int j = q * 4 + (lane >> 3);
                                rv[q] = (resid && c + j < nt)
                                            ? *reinterpret_cast<const float4*>(
                                                  resid + (row0 + n0 + c + j) * static_cast<int64_t>(a.ldr) + mbase + f)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int j = q * 4 + (lane >> 3);
                                if (c + j < nt) {
                                    float4 v = *reinterpret_cast<const float4*>(scr + j * 32 + f);
                                    v.x += rv[q].x; v.y += rv[q].y; v.z += rv[q].z; v.w += rv[q].w;
                                    *reinterpret_cast<float4*>(
                                        outp + (row0 + n0 + c + j) * static_cast<int64_t>(a.ldo) + mbase + f) = v;
                                }
                            }
                            __syncwarp();
                        } else {  // kEpiSiluPacked
                            uint16_t* sb = reinterpret_cast<uint16_t*>(scr);
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                sb[j * 32 + lane] =
                                    f32_to_bf16_bits(silu(__uint_as_float(r0[h][j])) * __uint_as_float(r1[h][j]));
                            __syncwarp();
                            const int f = (lane & 3) * 8;
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
                                const int j = q * 8 + (lane >> 2);
                                if (c + j < nt)
                                    *reinterpret_cast<uint4*>(a.out_packed + b_packed_off(row0 + n0 + c + j, mbase + f,
                                                                                          a.out_R)) =
                                        *reinterpret_cast<const uint4*>(sb + j * 32 + f);
                            }
                            __syncwarp();
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&ctl->tempty[acc]);
                if (++acc == acc_stages) { acc = 0; acc_phase ^= 1; }
            }
        }
    }
    if (tr && warp == 1 && lane == 0) tr[4] = globaltimer();  // all MMAs issued
    if (tr && warp == 2 && lane == 0) tr[6] = globaltimer();  // this warp's epilogue done
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, a.tmem_cols);
    }
    if (tr && threadIdx.x == 0) tr[7] = globaltimer();
    if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[1], ~globaltimer());
}

}  // namespace

int gemm_smem_bytes(int n_mats, int n_cap, int stages) {
    return stages * (n_mats * kATileBytes + n_cap * 128) + 1024 /*align*/ + kCtlBytes + kEpiScratch;
}

cudaError_t launch_gemm(GemmArgs a, int num_sms, cudaStream_t stream) {
    if (a.n_mats < 1 || a.n_mats > kMaxMats || a.K % kBlockK || a.n_cap % 16 || a.n_cap < 16 ||
        a.n_cap > 256 || a.R % 16 || a.n_chunks < 1 || a.k_splits < 1 ||
        a.k_splits > a.K / kBlockK || (a.k_splits > 1 && a.epi != kEpiF32) ||
        (a.epi == kEpiF32 && (a.ldo % 4 || a.ldr % 4 || a.split_stride % 4)))  // 16-byte epilogue stores
        return cudaErrorInvalidValue;
    const int per_stage = a.n_mats * kATileBytes + a.n_cap * 128;
    const int budget = 227 * 1024 - 1024 - kCtlBytes - kEpiScratch;
    a.stages = budget / per_stage;
    if (a.stages > 8) a.stages = 8;
    if (a.stages < 2) return cudaErrorInvalidValue;
    const int acc_cols = a.n_mats * a.n_cap;
    a.acc_stages = (2 * acc_cols <= 512) ? 2 : 1;
    int need = a.acc_stages * acc_cols;
    int cols = 32;
    while (cols < need) cols <<= 1;
    a.tmem_cols = cols;
    const int smem = gemm_smem_bytes(a.n_mats, a.n_cap, a.stages);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int n_virtual = a.G * a.RB * a.n_chunks * a.k_splits;
    const int grid = n_virtual < num_sms ? n_virtual : num_sms;
    if (grid <= 0) return cudaSuccess;
    gemm_tc_kernel<<<grid, kThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace mltk
