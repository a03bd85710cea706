// Register-decode GEMM for encoded weight tiles (GemmArgs::codec = 2, the
// "fragment-order" layout of runtime/weight_codec.hpp).
//
// Why a second engine.  The tcgen05 path (gemm_tc.cu, codec = 1) must expand
// each encoded tile back into a 16 KiB bf16 smem image before UMMA can read
// it: decoder warps load the tile, barrier, store it in place, fence the
// async proxy, barrier, and hand the stage to the MMA warp.  That chain sits
// inside every ring stage's round trip (land -> decode -> MMA -> release),
// and with 16 KiB slots only 4 stages fit, so the expert down GEMM streamed
// ~4 TB/s of encoded bytes (ktrace: 800 ns per 2-tile stage, 2.4 us
// issue-to-MMA) where HBM gives 6.5.  Here the tensor cores are fed from
// REGISTERS (mma.sync m16n8k16, ~550 TFLOP/s measured on this B200,
// tools/mma_probe.cu; the decode-time expert GEMMs need ~140): each thread
// decodes exactly its own A fragments, so nothing is written back, no proxy
// fence or cross-warp barrier sits in a stage, a stage is only the 12.4 KB
// encoded tile (+ the token tile), and the ring is 2x deeper.
//
// Fragment order: an encoded tile covers 128 weight rows x 64 k; its 8192
// bf16 are ordered so that 8-weight unit u = (m16 block mb, k16 block kk,
// lane) is lane's m16n8k16 A fragment {a0, a1, a2, a3} of rows 16mb + g /
// +8 and k 16kk + 2tg / +8 (g = lane/4, tg = lane%4).  Codec fields as in
// weight_codec.hpp: low bytes raw, high bytes as 4-bit codes into a 15-entry
// table, escapes listed by position.  A page-table entry with tag bit 0 is a
// raw fallback block (16 KiB bf16 tiles in the same fragment order).
//
// CTA: warp 0 = producer (1-D bulk copies of the encoded A tiles and the
// token tile into a multi-stage mbarrier ring), warps 1..8 = consumers; warp
// w owns m16 block w - 1 (16 weight rows) of the unit's 128, decodes its 4
// fragments per matrix and k-block into registers, and multiplies them with
// the token fragments (ldmatrix from the swizzled B tile) into fp32
// accumulators held in registers for up to 64 tokens.  Two CTAs per SM.
// Epilogue: fp32 rows (+ residual, or split-K partials) or the fused SiLU(g)*u
// into the packed operand of the down projection, like gemm_tc.
#include <cstdint>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kCWarps = 8;                    // consumer warps (m16 blocks of a 128-row tile)
constexpr int kCThreads = 32 * (kCWarps + 1);
// n8 token blocks per chunk held in registers: 64 tokens for one matrix, 32
// for gate/up (two accumulator sets; more tokens loop over chunks)
template <int NMATS>
constexpr int max_nb() { return NMATS == 2 ? 4 : 8; }
constexpr int kEncTile = 12432;               // encoded tile bytes (weight_codec.hpp)
constexpr int kRawTile = 16384;
constexpr int kMaxStagesC = 16;
constexpr int kMats = 2;

struct CtlC {
    uint64_t full[kMaxStagesC];
    uint64_t empty[kMaxStagesC];
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// One 8-weight unit: low bytes lo (8 B), codes cd (8 nibbles), table T ->
// the 8 bf16 (4 registers) in unit order.  Per 4 weights: two PRMT table
// lookups (codes 0-7 / 8-15), a sign-replicating PRMT turning each code's
// bit 3 into a byte mask, one select, two interleaving PRMTs.
__device__ __forceinline__ uint32_t hi4(uint32_t sel, uint32_t m, const uint4& T) {
    const uint32_t a = prmt(T.x, T.y, sel);
    const uint32_t b = prmt(T.z, T.w, sel);
    return (a & ~m) | (b & m);
}
__device__ __forceinline__ uint4 decode_unit(uint2 lo, uint32_t cd, const uint4& T) {
    const uint32_t c4 = cd << 4;
    const uint32_t h0 = hi4(cd & 0x7777u, prmt(c4, cd, 0xD9C8u), T);
    const uint32_t h1 = hi4((cd >> 16) & 0x7777u, prmt(c4, cd, 0xFBEAu), T);
    uint4 o;
    o.x = prmt(lo.x, h0, 0x5140u);
    o.y = prmt(lo.x, h0, 0x7362u);
    o.z = prmt(lo.y, h1, 0x5140u);
    o.w = prmt(lo.y, h1, 0x7362u);
    return o;
}

__device__ __forceinline__ const uint8_t* untag(const uint8_t* p, bool& raw) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    raw = (u & 1u) != 0;
    return reinterpret_cast<const uint8_t*>(u & ~static_cast<uintptr_t>(1));
}

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

struct Unit {
    int g, rb, c, kb0, kb1;
};
__device__ __forceinline__ Unit unit_of(const GemmArgs& a, int v, int KB) {
    Unit u;
    const int ks = v % a.k_splits, w = v / a.k_splits;
    u.c = w % a.n_chunks;
    u.g = (w / a.n_chunks) % a.G;
    u.rb = w / a.n_chunks / a.G;
    u.kb0 = ks * KB / a.k_splits;
    u.kb1 = (ks + 1) * KB / a.k_splits;
    return u;
}

template <int NMATS>
__global__ void __launch_bounds__(kCThreads, 2) gemm_codec_kernel(const GemmArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    // stage = [NMATS A slots | B tile of n_cap rows x 128 B]; a slot holds an
    // encoded tile (12432 B), or a raw fallback tile (16 KiB) when the caller
    // says some block of this GEMM is stored raw (GemmArgs::codec_raw)
    const int slot = a.codec_raw ? kRawTile : kEncTile;
    const int b_bytes = a.n_cap * 128;
    const int stage_bytes = NMATS * slot + b_bytes;
    const int stages = a.stages;
    CtlC* ctl = reinterpret_cast<CtlC*>(smem + stages * stage_bytes);
    const int warp = static_cast<int>(threadIdx.x) >> 5;
    const int lane = static_cast<int>(threadIdx.x) & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&ctl->full[s], 1);
            mbar_init(&ctl->empty[s], kCWarps);
        }
        fence_mbar_init();
    }
    pdl_trigger();
    __syncthreads();
    pdl_wait();
    if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[0], globaltimer());

    const int KB = a.K / kBlockK;
    const int n_units = a.G * a.RB * a.n_chunks * a.k_splits;

    if (warp == 0) {
        // ===== producer: encoded A tiles + token tile per k-block =====
        if (lane == 0) {
            const uint64_t pol_w = l2_evict_first(), pol_x = l2_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int v = blockIdx.x; v < n_units; v += gridDim.x) {
                const Unit u = unit_of(a, v, KB);
                const int rows = a.b_cnt ? a.b_cnt[u.g] : a.rows_dense;
                if (rows <= 0) continue;
                const int row0 = a.b_off ? a.b_off[u.g] : 0;
                const uint8_t* ab[NMATS];
                int tb[NMATS], tx = 0;
#pragma unroll
                for (int mt = 0; mt < NMATS; ++mt) {
                    bool raw;
                    ab[mt] = untag(a.a_table[(static_cast<int64_t>(mt) * a.G + u.g) * a.RB + u.rb], raw);
                    tb[mt] = raw ? kRawTile : kEncTile;
                    tx += tb[mt];
                }
                for (int n0 = u.c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                    const int nt = min(a.n_cap, rows - n0);
                    const int ntp = (nt + 7) & ~7;
                    for (int kb = u.kb0; kb < u.kb1; ++kb) {
                        mbar_wait(&ctl->empty[stage], phase ^ 1);
                        uint8_t* const st = smem + stage * stage_bytes;
                        mbar_expect_tx(&ctl->full[stage], tx + ntp * 128);
#pragma unroll
                        for (int mt = 0; mt < NMATS; ++mt)
                            bulk_g2s(st + mt * slot, ab[mt] + static_cast<int64_t>(kb) * tb[mt], tb[mt],
                                     &ctl->full[stage], pol_w);
                        bulk_g2s(st + NMATS * slot,
                                 a.b + static_cast<int64_t>(kb) * a.R * 128 + static_cast<int64_t>(row0 + n0) * 128,
                                 ntp * 128, &ctl->full[stage], pol_x);
                        if (++stage == stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else {
        // ===== consumers: decode own fragments, mma.sync, epilogue =====
        const int cw = warp - 1;          // m16 block of the 128-row tile
        const int g = lane >> 2, tg = lane & 3;
        // ldmatrix lane addressing for token (B) fragments: matrices (nb, c), (nb, c+1), (nb+1, c), (nb+1, c+1)
        const int mi = lane >> 3, rr = lane & 7;
        int stage = 0;
        uint32_t phase = 0;
        for (int v = blockIdx.x; v < n_units; v += gridDim.x) {
            const Unit u = unit_of(a, v, KB);
            const int rows = a.b_cnt ? a.b_cnt[u.g] : a.rows_dense;
            if (rows <= 0) continue;
            const int row0 = a.b_off ? a.b_off[u.g] : 0;
            bool raw[NMATS];
#pragma unroll
            for (int mt = 0; mt < NMATS; ++mt)
                untag(a.a_table[(static_cast<int64_t>(mt) * a.G + u.g) * a.RB + u.rb], raw[mt]);
            for (int n0 = u.c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                const int nt = min(a.n_cap, rows - n0);
                const int nb_used = (nt + 7) >> 3;
                constexpr int kMaxNB = max_nb<NMATS>();
                float acc[NMATS][kMaxNB][4];
#pragma unroll
                for (int mt = 0; mt < NMATS; ++mt)
#pragma unroll
                    for (int nb = 0; nb < kMaxNB; ++nb) acc[mt][nb][0] = acc[mt][nb][1] = acc[mt][nb][2] = acc[mt][nb][3] = 0.f;
                for (int kb = u.kb0; kb < u.kb1; ++kb) {
                    mbar_wait(&ctl->full[stage], phase);
                    const uint32_t st = smem_u32(smem + stage * stage_bytes);
                    const uint32_t sb = st + NMATS * slot;
                    // Every shared load of the stage first (this warp's 4 fragments per
                    // matrix, the tables, the escape list), then the decode + MMA chains:
                    // independent work in flight instead of one load latency per fragment.
                    uint4 T[NMATS];
                    uint2 lo[NMATS][4];
                    uint32_t cd[NMATS][4];
                    uint32_t esc[NMATS];  // this lane's escape entry {u16 idx, u8 hi} or ~0
#pragma unroll
                    for (int mt = 0; mt < NMATS; ++mt) {
                        const uint32_t ta = st + mt * slot;
                        if (!raw[mt]) {
                            T[mt] = lds128(ta + 12288);
                            const uint32_t n = lds32(ta + 12304) & 0xffffu;
                            esc[mt] = static_cast<uint32_t>(lane) < n ? lds32(ta + 12308 + 4 * lane) : ~0u;
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const int unit = (cw * 4 + kk) * 32 + lane;
                                lo[mt][kk] = lds64(ta + unit * 8);
                                cd[mt][kk] = lds32(ta + 8192 + unit * 4);
                            }
                        } else {
                            esc[mt] = ~0u;
                        }
                    }
                    // escapes that fall into this warp's fragments (weight index >> 10 = warp):
                    // one ballot per matrix and stage, the patch loop only when there are some
                    unsigned emask[NMATS];
#pragma unroll
                    for (int mt = 0; mt < NMATS; ++mt)
                        emask[mt] = __ballot_sync(0xffffffffu, esc[mt] != ~0u &&
                                                                   static_cast<int>((esc[mt] & 0xffffu) >> 10) == cw);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint4 A[NMATS];
#pragma unroll
                        for (int mt = 0; mt < NMATS; ++mt) {
                            if (raw[mt]) {
                                A[mt] = lds128(st + mt * slot + ((cw * 4 + kk) * 32 + lane) * 16);
                                continue;
                            }
                            A[mt] = decode_unit(lo[mt][kk], cd[mt][kk], T[mt]);
                            unsigned m = emask[mt];
                            while (m) {  // rare: high bytes outside the table
                                const int src = __ffs(m) - 1;
                                m &= m - 1;
                                const uint32_t e = __shfl_sync(0xffffffffu, esc[mt], src);
                                const uint32_t idx = e & 0xffffu, hi = (e >> 16) & 0xffu;
                                if (static_cast<int>((idx >> 8) & 3u) == kk && static_cast<int>((idx >> 3) & 31u) == lane) {
                                    const uint32_t j = idx & 7u;  // weight j of the unit: reg j/2, byte 2(j&1)+1
                                    const uint32_t sh = ((j & 1u) * 2u + 1u) * 8u;
                                    const uint32_t keep = ~(0xffu << sh), put = hi << sh, q = j >> 1;
                                    if (q == 0) A[mt].x = (A[mt].x & keep) | put;
                                    else if (q == 1) A[mt].y = (A[mt].y & keep) | put;
                                    else if (q == 2) A[mt].z = (A[mt].z & keep) | put;
                                    else A[mt].w = (A[mt].w & keep) | put;
                                }
                            }
                        }
#pragma unroll
                        for (int nb = 0; nb < kMaxNB; nb += 2) {
                            if (nb >= nb_used) break;
                            // token rows nb*8.. (+8 for the second pair), k chunks 2kk, 2kk+1
                            const int row = (nb + (mi >> 1)) * 8 + rr;
                            const int ch = 2 * kk + (mi & 1);
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4(sb + row * 128 + ((ch ^ rr) << 4), b0, b1, b2, b3);
#pragma unroll
                            for (int mt = 0; mt < NMATS; ++mt) {
                                mma16816(acc[mt][nb], A[mt], b0, b1);
                                if (nb + 1 < nb_used) mma16816(acc[mt][nb + 1], A[mt], b2, b3);
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&ctl->empty[stage]);
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
                // ---- epilogue: acc[mt][nb] = (rows g / g+8) x (tokens 2tg, 2tg+1) of n8 block nb ----
                const int ks = v % a.k_splits;
                const int mbase = u.rb * kBlockM + cw * 16;
                if (a.epi == kEpiF32) {
                    float* const outp = a.out_f32 + static_cast<int64_t>(ks) * a.split_stride;
                    const float* const resid = a.k_splits == 1 ? a.residual : nullptr;
#pragma unroll
                    for (int nb = 0; nb < kMaxNB; ++nb) {
                        if (nb >= nb_used) break;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int tok = nb * 8 + 2 * tg + (e & 1);
                            const int m = mbase + g + (e >> 1) * 8;
                            if (tok < nt) {
                                const int64_t r = row0 + n0 + tok;
                                float val = acc[0][nb][e] * a.alpha;
                                if (resid) val += resid[r * a.ldr + m];
                                outp[r * a.ldo + m] = val;
                            }
                        }
                    }
                } else if constexpr (NMATS == 2) {  // SiLU(g) * u -> packed bf16 operand of the down GEMM
#pragma unroll
                    for (int nb = 0; nb < kMaxNB; ++nb) {
                        if (nb >= nb_used) break;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int tok = nb * 8 + 2 * tg + (e & 1);
                            const int m = mbase + g + (e >> 1) * 8;
                            if (tok < nt)
                                *reinterpret_cast<uint16_t*>(a.out_packed + b_packed_off(row0 + n0 + tok, m, a.out_R)) =
                                    f32_to_bf16_bits(silu(acc[0][nb][e]) * acc[1][nb][e]);
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[1], ~globaltimer());
}

}  // namespace

int gemm_codec_smem_bytes(int n_mats, int n_cap, int stages, bool raw_slots) {
    return stages * (n_mats * (raw_slots ? kRawTile : kEncTile) + n_cap * 128) + 1024 + static_cast<int>(sizeof(CtlC));
}

cudaError_t launch_gemm_codec(GemmArgs a, int num_sms, cudaStream_t stream) {
    if (a.n_mats < 1 || a.n_mats > kMats || a.K % kBlockK || a.n_cap < 16 ||
        a.n_cap > 8 * (a.n_mats == 2 ? max_nb<2>() : max_nb<1>()) || a.n_cap % 16 ||
        a.R % 16 || a.n_chunks < 1 || a.k_splits < 1 || a.k_splits > a.K / kBlockK ||
        (a.k_splits > 1 && a.epi != kEpiF32) || (a.epi == kEpiSiluPacked && a.n_mats != 2) ||
        (a.epi == kEpiF32 && a.n_mats != 1))
        return cudaErrorInvalidValue;
    // two CTAs per SM: each gets half of the 227 KiB (ring + control)
    const int per_stage = a.n_mats * (a.codec_raw ? kRawTile : kEncTile) + a.n_cap * 128;
    a.stages = (227 * 1024 / 2 - 1024 - static_cast<int>(sizeof(CtlC))) / per_stage;
    if (a.stages > kMaxStagesC) a.stages = kMaxStagesC;
    if (a.stages < 2) return cudaErrorInvalidValue;
    const int smem = gemm_codec_smem_bytes(a.n_mats, a.n_cap, a.stages, a.codec_raw != 0);
    const void* kern = a.n_mats == 2 ? reinterpret_cast<const void*>(gemm_codec_kernel<2>)
                                     : reinterpret_cast<const void*>(gemm_codec_kernel<1>);
    if (cudaError_t e = ensure_smem_attr(kern, smem); e != cudaSuccess) return e;
    const int units = a.G * a.RB * a.n_chunks * a.k_splits;
    const int grid = units < 2 * num_sms ? units : 2 * num_sms;
    if (grid <= 0) return cudaSuccess;
    return a.n_mats == 2 ? launch_k(gemm_codec_kernel<2>, dim3(grid), dim3(kCThreads), smem, stream, a)
                         : launch_k(gemm_codec_kernel<1>, dim3(grid), dim3(kCThreads), smem, stream, a);
}

}  // namespace mltk
