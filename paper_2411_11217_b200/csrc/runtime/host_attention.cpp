// Host-core GQA decode attention — the paper's default placement (A_g = 0,
// PAPER.md:390-392 "CPU attention = the softmax part", 553 "customized CPU
// GQA kernels").  It is a policy choice, not a fallback: the task is
// TaskKind::CpuAttn on Resource::Cpu of the CGOPipe DAG.
//
// Input: the D1 offload of one micro-batch (bf16 rows q|k|v, roped).  The
// new k/v are appended to the host KV cache, laid out head-major
// [layer][seq][kv_head][ctx][d] so each (seq, head) is one contiguous stream
// for the hardware prefetcher.  One work item per (seq, kv head) computes all
// G = n_q/n_kv query heads against one pass over K and V (GQA reuse): on the
// AMX tile unit where the host has it (gqa_item_amx), else with AVX-512
// (VDPBF16PS scores, fp32 FMA P.V).  Output is written straight in the packed
// operand layout of the O projection, so the D2 upload needs no device-side
// repack.  The team is pinned to the cores host_cores() leaves to attention.
// Measured on the GPU box's 16 host cores (tools/host_gqa_probe.py, 8x7B
// shape, 256 sequences x ctx 520): 3.6 ms per layer on 14 cores = 149 GB/s
// of KV (the cores' plain read stream: 207 GB/s); the AVX-512 path 3.8 ms,
// the previous per-head loop order ~5 ms.
#include <immintrin.h>
#include <omp.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <utility>
#include <cmath>
#include <cstring>
#include <vector>

#include "../kernels/common.cuh"
#include "host_gqa.hpp"
#include "host_layout.hpp"
#include "runtime.hpp"

namespace mlt {

namespace {

inline __m512 load_bf16x16(const uint16_t* p) {
    const __m256i raw = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p));
    return _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(raw), 16));
}

constexpr int kD = 128;
constexpr int kMaxG = 16;

// e^x for x <= 0 (softmax arguments), 16 lanes: n = round(x / ln 2), f = x -
// n ln 2 (Cody-Waite, two-part ln 2), e^f by its degree-6 Taylor polynomial
// (|f| <= 0.35: rel. error ~2e-7), scaled by 2^n (VSCALEFPS).
inline __m512 exp16(__m512 x) {
    x = _mm512_max_ps(x, _mm512_set1_ps(-87.0f));
    const __m512 n = _mm512_roundscale_ps(_mm512_mul_ps(x, _mm512_set1_ps(1.4426950408889634f)),
                                          _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    __m512 f = _mm512_fnmadd_ps(n, _mm512_set1_ps(0.693145751953125f), x);  // ln 2 high part (exact n*hi)
    f = _mm512_fnmadd_ps(n, _mm512_set1_ps(1.428606765330187e-06f), f);    // ln 2 low part
    __m512 p = _mm512_set1_ps(1.0f / 720.0f);
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f / 120.0f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f / 24.0f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f / 6.0f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(0.5f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f));
    return _mm512_scalef_ps(p, n);
}

// r[i] = sum of the 16 lanes of a[i], i = 0..15 (transpose-add tree, 45 ops
// instead of 16 horizontal reductions)
__attribute__((target("avx512f"))) inline __m512 hsum16(__m512 (&a)[16]) {
    __m512 b[8], c[4], e[2];
    for (int k = 0; k < 8; ++k)
        b[k] = _mm512_add_ps(_mm512_unpacklo_ps(a[2 * k], a[2 * k + 1]), _mm512_unpackhi_ps(a[2 * k], a[2 * k + 1]));
    for (int k = 0; k < 4; ++k)
        c[k] = _mm512_add_ps(_mm512_shuffle_ps(b[2 * k], b[2 * k + 1], 0x44), _mm512_shuffle_ps(b[2 * k], b[2 * k + 1], 0xEE));
    for (int k = 0; k < 2; ++k)
        e[k] = _mm512_add_ps(_mm512_shuffle_f32x4(c[2 * k], c[2 * k + 1], 0x88),
                             _mm512_shuffle_f32x4(c[2 * k], c[2 * k + 1], 0xDD));
    return _mm512_add_ps(_mm512_shuffle_f32x4(e[0], e[1], 0x88), _mm512_shuffle_f32x4(e[0], e[1], 0xDD));
}

// Scores of 16 consecutive keys for one head with AVX512-BF16 dot products:
// acc_j = sum over 4 x 32 bf16 pairs of q . k_j (fp32 accumulate), reduced by
// the tree above.  Keys past n contribute zero rows (never read).
__attribute__((target("avx512f,avx512bf16"))) inline __m512 scores16_bf16(const __m512bh (&q)[4],
                                                                         const uint16_t* k, int n) {
    __m512 acc[16];
    for (int j = 0; j < 16; ++j) {
        acc[j] = _mm512_setzero_ps();
        if (j < n) {
            const uint16_t* kr = k + static_cast<size_t>(j) * kD;
            for (int c = 0; c < 4; ++c)
                acc[j] = _mm512_dpbf16_ps(acc[j], q[c], (__m512bh)_mm512_loadu_si512(kr + 32 * c));
        }
    }
    return hsum16(acc);
}


// P.V for one (sequence, kv head), G query heads, register-blocked: every
// 64-byte V load is split into its even and odd bf16 lanes as fp32 (shift /
// mask, no widening), and a pass keeps G x kU accumulators of 32 dims in
// registers (kU = 32-dim units per pass, sized so G * 2kU accumulators + 2kU
// values + the broadcast fit the 32 zmm registers).  V is read once from
// DRAM: the passes touch disjoint 64-byte columns of each 256-byte row.
// Lane order inside a 32-dim unit is (even dims, odd dims); un-permuted at
// the store.
template <int G>
__attribute__((target("avx512f,avx512bw,avx512bf16"))) void pv_pass(const uint16_t* vc, int L, const float* sc,
                                                                      int ldsc, const float* inv, uint16_t* out) {
    constexpr int kU = G <= 3 ? 4 : G <= 6 ? 2 : 1;  // 32-dim units per pass
    const __m512i hi_mask = _mm512_set1_epi32(static_cast<int>(0xFFFF0000u));
    for (int u0 = 0; u0 < kD / 32; u0 += kU) {
        __m512 o[G][2 * kU];
        for (int g = 0; g < G; ++g)
            for (int c = 0; c < 2 * kU; ++c) o[g][c] = _mm512_setzero_ps();
        const uint16_t* vp = vc + u0 * 32;
        for (int j = 0; j < L; ++j, vp += kD) {
            __m512 v[2 * kU];
            for (int u = 0; u < kU; ++u) {
                const __m512i x = _mm512_loadu_si512(vp + 32 * u);
                v[2 * u] = _mm512_castsi512_ps(_mm512_slli_epi32(x, 16));          // even dims
                v[2 * u + 1] = _mm512_castsi512_ps(_mm512_and_si512(x, hi_mask));  // odd dims
            }
            for (int g = 0; g < G; ++g) {
                const __m512 pj = _mm512_set1_ps(sc[static_cast<size_t>(g) * ldsc + j]);
                for (int c = 0; c < 2 * kU; ++c) o[g][c] = _mm512_fmadd_ps(pj, v[c], o[g][c]);
            }
        }
        for (int g = 0; g < G; ++g) {
            const __m512 s = _mm512_set1_ps(inv[g]);
            for (int u = 0; u < kU; ++u) {
                const __m512 ev = _mm512_mul_ps(o[g][2 * u], s), od = _mm512_mul_ps(o[g][2 * u + 1], s);
                // interleave back to dim order: (e0 o0 e1 o1 ...) over 32 dims
                const __m512 lo = _mm512_unpacklo_ps(ev, od), hi = _mm512_unpackhi_ps(ev, od);
                const __m512 d0 = _mm512_permutex2var_ps(lo, _mm512_setr_epi32(0, 1, 2, 3, 16, 17, 18, 19, 4, 5, 6, 7, 20, 21, 22, 23), hi);
                const __m512 d1 = _mm512_permutex2var_ps(lo, _mm512_setr_epi32(8, 9, 10, 11, 24, 25, 26, 27, 12, 13, 14, 15, 28, 29, 30, 31), hi);
                // RNE fp32 -> bf16 (VCVTNE2PS2BF16: d1 to the high half)
                const __m512bh pk = _mm512_cvtne2ps_pbh(d1, d0);
                _mm512_storeu_si512(out + static_cast<size_t>(g) * kD + (u0 + u) * 32, (__m512i)pk);
            }
        }
    }
}

using PvFn = void (*)(const uint16_t*, int, const float*, int, const float*, uint16_t*);
template <int... Gs>
constexpr PvFn pv_for(int G, std::integer_sequence<int, Gs...>) {
    PvFn f = nullptr;
    ((G == Gs + 1 ? (f = &pv_pass<Gs + 1>, 0) : 0), ...);
    return f;
}

// ---- AMX path (Sapphire Rapids and later: AMX-TILE + AMX-BF16) ----------
// Both products of one (sequence, kv head) on the tile unit, so the item is
// bound by the DRAM stream of K and V rather than by the AVX-512 FMA ports:
//   scores  S[16 keys][G] += K[16 keys][32 dims] . Qt[16 dim pairs][G x 2]
//           (A = 16 cache rows straight from the K stream, B = q in VNNI
//           pairs, built once per item), 4 TDPBF16PS per 16 keys;
//   output  O[G][16 dims] += P[G][32 keys] . Vt[16 key pairs][16 x 2]
//           (A = bf16 softmax numerators, B = two V rows interleaved by
//           VPUNPCK{L,H}WD on the fly; the lane shuffle permutes the output
//           columns, undone once per item), 4 tiles = 64 dims per pass,
//           2 passes (disjoint 128-byte halves of each V row).
// P enters the second product as two bf16 terms, P = hi + lo (hi = bf16(P),
// lo = bf16(P - hi)), two TDPBF16PS per block: ~16 mantissa bits, so the
// result tracks the fp32 AVX-512 path (V is exact in bf16); scores, max, exp
// and the denominator stay fp32.
struct alignas(64) TileCfg {
    uint8_t palette = 1, start_row = 0;
    uint8_t reserved[14] = {};
    uint16_t colsb[16] = {};
    uint8_t rows[16] = {};
};

bool amx_request() {
    unsigned a, b, c, d;
    __asm__ volatile("cpuid" : "=a"(a), "=b"(b), "=c"(c), "=d"(d) : "a"(7), "c"(0));
    const bool tile = (d >> 24) & 1u, bf16 = (d >> 22) & 1u;
    if (!tile || !bf16) return false;
    constexpr long kArchReqXcompPerm = 0x1023, kXfeatureXtiledata = 18;
    return syscall(SYS_arch_prctl, kArchReqXcompPerm, kXfeatureXtiledata) == 0;
}

std::atomic<int> g_amx_mode{-1};  // -1: undecided, 0: off, 1: on

__attribute__((target("avx512f,avx512bw,avx512bf16,amx-tile,amx-bf16"))) void gqa_item_amx(
    const uint16_t* q, const uint16_t* kc, const uint16_t* vc, int L, int G, float scale, float* sc, int ldsc,
    uint16_t* out) {
    // scratch carve-up (host_gqa_scratch_floats)
    uint16_t* pbf = reinterpret_cast<uint16_t*>(sc + static_cast<size_t>(kMaxG) * ldsc);  // [G][ldsc] bf16 hi
    uint16_t* plo = pbf + static_cast<size_t>(kMaxG) * ldsc;                                // [G][ldsc] bf16 lo
    float* ex = sc + static_cast<size_t>(kMaxG) * ldsc * 2;
    ex = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ex) + 63) & ~uintptr_t(63));
    uint32_t* qb = reinterpret_cast<uint32_t*>(ex);              // [4][16][16] words
    float* sbuf = ex + 1024;                                     // [2][16][16]
    uint16_t* ktail = reinterpret_cast<uint16_t*>(ex + 1536);    // [16][128]
    uint16_t* vb = reinterpret_cast<uint16_t*>(ex + 2560);       // [4][16][32]
    float* obuf = ex + 3584;                                     // [16][64]

    // ---- scores ----
    TileCfg ck;
    ck.rows[0] = 16, ck.colsb[0] = static_cast<uint16_t>(4 * G);  // S
    ck.rows[1] = 16, ck.colsb[1] = 64;                            // K chunk
    for (int t = 2; t < 6; ++t) ck.rows[t] = 16, ck.colsb[t] = static_cast<uint16_t>(4 * G);  // Qt chunks
    ck.rows[6] = 16, ck.colsb[6] = static_cast<uint16_t>(4 * G);  // S, second block
    ck.rows[7] = 16, ck.colsb[7] = 64;                            // K chunk, second block
    _tile_loadconfig(&ck);
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(q);
    for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 16; ++r)
            for (int n = 0; n < G; ++n) qb[(c * 16 + r) * 16 + n] = q32[n * (kD / 2) + 16 * c + r];
    _tile_loadd(2, qb, 64);
    _tile_loadd(3, qb + 256, 64);
    _tile_loadd(4, qb + 512, 64);
    _tile_loadd(5, qb + 768, 64);
    const __m512i rows16 = _mm512_mullo_epi32(_mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15),
                                              _mm512_set1_epi32(16));
    __m512 m16[kMaxG];
    for (int g = 0; g < G; ++g) m16[g] = _mm512_set1_ps(-INFINITY);
    const __m512 vscale = _mm512_set1_ps(scale);
    // two 16-key blocks per iteration on two accumulators (S: tmm0 / tmm6,
    // K chunk: tmm1 / tmm7), so the tile unit overlaps the two dependency
    // chains of 4 TDPBF16PS
    auto scores_out = [&](const float* sb, int j, int n) {
        const __mmask16 live = static_cast<__mmask16>((1u << n) - 1u);
        for (int g = 0; g < G; ++g) {
            const __m512 s16 = _mm512_mask_mul_ps(_mm512_set1_ps(-INFINITY), live,
                                                  _mm512_i32gather_ps(rows16, sb + g, 4), vscale);
            _mm512_storeu_ps(sc + static_cast<size_t>(g) * ldsc + j, s16);
            m16[g] = _mm512_max_ps(m16[g], s16);
        }
    };
    for (int j0 = 0; j0 < L; j0 += 32) {
        const int na = std::min(16, L - j0), nb = std::max(0, std::min(16, L - j0 - 16));
        const uint16_t* ka = kc + static_cast<size_t>(j0) * kD;
        const uint16_t* kb = ka + 16 * kD;
        // rows past L may lie past the stream: stage a partial block, zero-padded
        const int part = na < 16 ? na : nb;
        if (part > 0 && part < 16) {
            const uint16_t* src = na < 16 ? ka : kb;
            std::memcpy(ktail, src, static_cast<size_t>(part) * kD * 2);
            std::memset(ktail + part * kD, 0, static_cast<size_t>(16 - part) * kD * 2);
            (na < 16 ? ka : kb) = ktail;
        }
        _tile_zero(0);
        _tile_loadd(1, ka, kD * 2);
        if (nb) {
            _tile_zero(6);
            _tile_loadd(7, kb, kD * 2);
        }
        _tile_dpbf16ps(0, 1, 2);
        if (nb) _tile_dpbf16ps(6, 7, 2);
        _tile_loadd(1, ka + 32, kD * 2);
        if (nb) _tile_loadd(7, kb + 32, kD * 2);
        _tile_dpbf16ps(0, 1, 3);
        if (nb) _tile_dpbf16ps(6, 7, 3);
        _tile_loadd(1, ka + 64, kD * 2);
        if (nb) _tile_loadd(7, kb + 64, kD * 2);
        _tile_dpbf16ps(0, 1, 4);
        if (nb) _tile_dpbf16ps(6, 7, 4);
        _tile_loadd(1, ka + 96, kD * 2);
        if (nb) _tile_loadd(7, kb + 96, kD * 2);
        _tile_dpbf16ps(0, 1, 5);
        if (nb) _tile_dpbf16ps(6, 7, 5);
        _tile_stored(0, sbuf, 64);
        if (nb) _tile_stored(6, sbuf + 256, 64);
        scores_out(sbuf, j0, na);
        if (nb) scores_out(sbuf + 256, j0 + 16, nb);
    }
    // ---- softmax numerators: fp32 sum, P as bf16 hi + lo (zero past L to a 32-key block) ----
    float inv[kMaxG];
    const int L32 = (L + 31) & ~31;
    for (int g = 0; g < G; ++g) {
        const float* srow = sc + static_cast<size_t>(g) * ldsc;
        uint16_t* prow = pbf + static_cast<size_t>(g) * ldsc;
        uint16_t* lrow = plo + static_cast<size_t>(g) * ldsc;
        const __m512 m = _mm512_set1_ps(_mm512_reduce_max_ps(m16[g]));
        __m512 d16 = _mm512_setzero_ps();
        for (int j0 = 0; j0 < L32; j0 += 16) {
            __m512 e = _mm512_setzero_ps();
            if (j0 < L) {
                const int n = std::min(16, L - j0);
                const __mmask16 live = static_cast<__mmask16>((1u << n) - 1u);
                e = _mm512_maskz_mov_ps(live, exp16(_mm512_sub_ps(_mm512_loadu_ps(srow + j0), m)));
                d16 = _mm512_add_ps(d16, e);
            }
            const __m256bh hi = _mm512_cvtneps_pbh(e);
            const __m512 hf = _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32((__m256i)hi), 16));
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(prow + j0), (__m256i)hi);
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(lrow + j0), (__m256i)_mm512_cvtneps_pbh(_mm512_sub_ps(e, hf)));
        }
        inv[g] = 1.0f / _mm512_reduce_add_ps(d16);
    }
    // ---- P.V ----
    TileCfg cv;
    for (int t = 0; t < 4; ++t) cv.rows[t] = static_cast<uint8_t>(G), cv.colsb[t] = 64;  // O blocks
    cv.rows[4] = static_cast<uint8_t>(G), cv.colsb[4] = 64;                            // P
    cv.rows[5] = 16, cv.colsb[5] = 64;                                                  // Vt
    cv.rows[6] = 16, cv.colsb[6] = 64;
    cv.rows[7] = static_cast<uint8_t>(G), cv.colsb[7] = 64;                            // P lo
    _tile_loadconfig(&cv);
    for (int pass = 0; pass < 2; ++pass) {
        _tile_zero(0);
        _tile_zero(1);
        _tile_zero(2);
        _tile_zero(3);
        for (int j0 = 0; j0 < L; j0 += 32) {
            for (int r = 0; r < 16; ++r) {
                const int ja = j0 + 2 * r, jb = ja + 1;
                const uint16_t* va = vc + static_cast<size_t>(ja) * kD + 64 * pass;
                const uint16_t* vb2 = vc + static_cast<size_t>(jb) * kD + 64 * pass;
                for (int h = 0; h < 2; ++h) {
                    const __m512i a = ja < L ? _mm512_loadu_si512(va + 32 * h) : _mm512_setzero_si512();
                    const __m512i b = jb < L ? _mm512_loadu_si512(vb2 + 32 * h) : _mm512_setzero_si512();
                    _mm512_store_si512(vb + ((2 * h) * 16 + r) * 32, _mm512_unpacklo_epi16(a, b));
                    _mm512_store_si512(vb + ((2 * h + 1) * 16 + r) * 32, _mm512_unpackhi_epi16(a, b));
                }
            }
            _tile_loadd(4, pbf + j0, ldsc * 2);
            _tile_loadd(7, plo + j0, ldsc * 2);
            _tile_loadd(5, vb, 64);
            _tile_dpbf16ps(0, 4, 5);
            _tile_dpbf16ps(0, 7, 5);
            _tile_loadd(6, vb + 512, 64);
            _tile_dpbf16ps(1, 4, 6);
            _tile_dpbf16ps(1, 7, 6);
            _tile_loadd(5, vb + 1024, 64);
            _tile_dpbf16ps(2, 4, 5);
            _tile_dpbf16ps(2, 7, 5);
            _tile_loadd(6, vb + 1536, 64);
            _tile_dpbf16ps(3, 4, 6);
            _tile_dpbf16ps(3, 7, 6);
        }
        _tile_stored(0, obuf, 256);
        _tile_stored(1, obuf + 16, 256);
        _tile_stored(2, obuf + 32, 256);
        _tile_stored(3, obuf + 48, 256);
        // block b = 2h + (lo|hi), column n -> dim 32h + 8(n/4) + 4(b%2) + n%4 of this pass's 64
        for (int g = 0; g < G; ++g) {
            alignas(64) float o[64];
            for (int b = 0; b < 4; ++b)
                for (int nn = 0; nn < 16; ++nn)
                    o[32 * (b / 2) + 8 * (nn / 4) + 4 * (b % 2) + nn % 4] = obuf[g * 64 + 16 * b + nn] * inv[g];
            for (int u = 0; u < 2; ++u) {
                const __m512bh pk = _mm512_cvtne2ps_pbh(_mm512_load_ps(o + 32 * u + 16), _mm512_load_ps(o + 32 * u));
                _mm512_storeu_si512(out + static_cast<size_t>(g) * kD + 64 * pass + 32 * u, (__m512i)pk);
            }
        }
    }
}

}  // namespace

bool host_gqa_amx() {
    int m = g_amx_mode.load();
    if (m < 0) {
        const char* env = std::getenv("MLT_HOST_AMX");
        const bool want = !(env && env[0] == '0');
        m = want && amx_request() ? 1 : 0;
        int expect = -1;
        if (!g_amx_mode.compare_exchange_strong(expect, m)) m = expect;
    }
    return m == 1;
}

bool host_gqa_set_amx(bool enable) {
    if (enable) {
        g_amx_mode.store(-1);
        return host_gqa_amx();
    }
    g_amx_mode.store(0);
    return false;
}

size_t host_gqa_scratch_floats(int max_ctx) {
    return static_cast<size_t>(kMaxG) * host_gqa_ldsc(max_ctx) * 2 + 4608 + 16;
}

int host_gqa_ldsc(int max_ctx) { return (max_ctx + 31) & ~31; }

namespace {
}  // namespace

bool host_gqa_bf16dot() {
    static const bool has = __builtin_cpu_supports("avx512bf16");
    return has;
}

// Scores, softmax numerators and P.V for one (sequence, kv head).  The K
// pass walks 16-key blocks and computes all G heads per block while the
// block (4 KiB) is in L1, so K streams from DRAM once; the V pass is pv_pass.
__attribute__((target("avx512f,avx512bw,avx512bf16"))) void host_gqa_item(
    const uint16_t* q, const uint16_t* kc, const uint16_t* vc, int L, int G, float scale, float* sc, int ldsc,
    uint16_t* out) {
    if (host_gqa_amx()) return gqa_item_amx(q, kc, vc, L, G, scale, sc, ldsc, out);
    float mx[kMaxG], inv[kMaxG];
    __m512 m16[kMaxG];
    for (int g = 0; g < G; ++g) m16[g] = _mm512_set1_ps(-INFINITY);
    if (host_gqa_bf16dot()) {
        // 4 VDPBF16PS per key and head (q and k stay bf16, fp32 accumulate),
        // one transpose-add tree per 16 keys and head
        for (int j0 = 0; j0 < L; j0 += 16) {
            const int n = std::min(16, L - j0);
            const __mmask16 live = static_cast<__mmask16>((1u << n) - 1u);
            const uint16_t* kb = kc + static_cast<size_t>(j0) * kD;
            for (int g = 0; g < G; ++g) {
                __m512bh qb[4];
                for (int c = 0; c < 4; ++c) qb[c] = (__m512bh)_mm512_loadu_si512(q + g * kD + 32 * c);
                const __m512 s16 = _mm512_mask_mov_ps(_mm512_set1_ps(-INFINITY), live,
                                                      _mm512_mul_ps(scores16_bf16(qb, kb, n), _mm512_set1_ps(scale)));
                _mm512_storeu_ps(sc + static_cast<size_t>(g) * ldsc + j0, s16);
                m16[g] = _mm512_max_ps(m16[g], s16);
            }
        }
    } else {
        __m512 qf[kMaxG][kD / 16];
        for (int g = 0; g < G; ++g)
            for (int c = 0; c < kD / 16; ++c)
                qf[g][c] = _mm512_mul_ps(load_bf16x16(q + g * kD + c * 16), _mm512_set1_ps(scale));
        for (int j = 0; j < L; ++j) {
            __m512 k[kD / 16];
            for (int c = 0; c < kD / 16; ++c) k[c] = load_bf16x16(kc + static_cast<size_t>(j) * kD + c * 16);
            for (int g = 0; g < G; ++g) {
                __m512 acc = _mm512_mul_ps(qf[g][0], k[0]);
                for (int c = 1; c < kD / 16; ++c) acc = _mm512_fmadd_ps(qf[g][c], k[c], acc);
                sc[static_cast<size_t>(g) * ldsc + j] = _mm512_reduce_add_ps(acc);
            }
        }
        for (int g = 0; g < G; ++g) {  // pad the tail block like the bf16 path
            for (int j = L; j < ((L + 15) & ~15); ++j) sc[static_cast<size_t>(g) * ldsc + j] = -INFINITY;
            for (int j0 = 0; j0 < L; j0 += 16)
                m16[g] = _mm512_max_ps(m16[g], _mm512_loadu_ps(sc + static_cast<size_t>(g) * ldsc + j0));
        }
    }
    for (int g = 0; g < G; ++g) mx[g] = _mm512_reduce_max_ps(m16[g]);
    for (int g = 0; g < G; ++g) {  // vectorised softmax numerators (tail lanes -> 0)
        float* srow = sc + static_cast<size_t>(g) * ldsc;
        const __m512 m = _mm512_set1_ps(mx[g]);
        __m512 d16 = _mm512_setzero_ps();
        for (int j0 = 0; j0 < L; j0 += 16) {
            const int n = std::min(16, L - j0);
            const __mmask16 live = static_cast<__mmask16>((1u << n) - 1u);
            const __m512 e = _mm512_maskz_mov_ps(live, exp16(_mm512_sub_ps(_mm512_loadu_ps(srow + j0), m)));
            _mm512_storeu_ps(srow + j0, e);
            d16 = _mm512_add_ps(d16, e);
        }
        inv[g] = 1.0f / _mm512_reduce_add_ps(d16);
    }
    static constexpr PvFn kPv[kMaxG] = {pv_for(1, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(2, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(3, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(4, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(5, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(6, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(7, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(8, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(9, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(10, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(11, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(12, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(13, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(14, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(15, std::make_integer_sequence<int, kMaxG>{}),
                                        pv_for(16, std::make_integer_sequence<int, kMaxG>{})};
    kPv[G - 1](vc, L, sc, ldsc, inv, out);
}

void Runtime::host_attention(int l, int mb, int step) {
    const int G = nq_ / nkv_;
    const int t0 = mb * mu_;
    const uint16_t* qkv = h_qkv_ + static_cast<size_t>(mb) * mu_ * W_;
    uint8_t* out = h_attn_ + static_cast<size_t>(mb) * Rmu_ * Ho_ * 2;  // this rank's heads
    const int32_t* pos = step_pos_.data() + static_cast<size_t>(step - 1) * N_;
    const float scale = 1.0f / std::sqrt(static_cast<float>(kD));
    // The team runs on the attention cores of host_cores(), one thread per
    // core: a launcher thread sharing a core with an attention thread would
    // either leave the GPU idle between the kernels of a PostAttn or stall
    // the team's closing barrier behind a preempted item.
    if (host_cores_.attn.empty()) host_cores_ = host_cores(shard_.rank, opt_.tp_shard_only ? 1 : shard_.size);
    const std::vector<int>& cores = host_cores_.attn;
    const int threads = opt_.host_threads > 0 ? opt_.host_threads : static_cast<int>(cores.size());
    const bool pin = host_cores_.pinned && threads <= static_cast<int>(cores.size());
    const int ldsc = host_gqa_ldsc(max_ctx_);
#pragma omp parallel num_threads(threads)
    {
        std::vector<float> sc(host_gqa_scratch_floats(max_ctx_));
        alignas(64) uint16_t ob[kMaxG * kD];
        if (pin) {
            thread_local int on_core = -1;
            const int c = cores[omp_get_thread_num()];
            if (on_core != c) pin_thread({c}), on_core = c;
        }
#pragma omp for collapse(2) schedule(dynamic, 1)
        for (int t = 0; t < mu_; ++t)
            for (int h = 0; h < nkv_; ++h) {
                const int seq = t0 + t;
                const int p = pos[seq];
                const uint16_t* row = qkv + static_cast<size_t>(t) * W_;
                const size_t base = ((static_cast<size_t>(l) * N_ + seq) * nkv_ + h) * max_ctx_;
                uint16_t* kc = h_kcache_ + base * kD;
                uint16_t* vc = h_vcache_ + base * kD;
                std::memcpy(kc + static_cast<size_t>(p) * kD, row + (nq_ + h) * kD, kD * 2);
                std::memcpy(vc + static_cast<size_t>(p) * kD, row + (nq_ + nkv_ + h) * kD, kD * 2);
                host_gqa_item(row + h * G * kD, kc, vc, p + 1, G, scale, sc.data(), ldsc, ob);
                for (int g = 0; g < G; ++g) {
                    const int col = (h * G + g) * kD;
                    for (int i = 0; i < kD; i += 8)
                        std::memcpy(out + mltk::b_packed_off(t, col + i, Rmu_), ob + g * kD + i, 16);
                }
            }
    }
}

HostCores host_cores(int rank, int sharing) {
    HostCores hc;
    cpu_set_t set;
    CPU_ZERO(&set);
    std::vector<int> all;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) {
        for (int c = 0; c < CPU_SETSIZE; ++c)
            if (CPU_ISSET(c, &set)) all.push_back(c);
    }
    if (all.empty())
        for (int c = 0; c < omp_get_num_procs(); ++c) all.push_back(c);
    if (all.size() < 4) {
        hc.attn = all;
        return hc;
    }
    static const int nl = [] {
        const char* e = std::getenv("MLT_LAUNCH_CORES");
        const int v = e ? std::atoi(e) : 2;
        return v < 1 ? 1 : v > 4 ? 4 : v;
    }();
    hc.launch.assign(all.begin(), all.begin() + nl);
    const int per = std::max(1, static_cast<int>(all.size() - nl) / std::max(1, sharing));
    const int first = nl + (rank % std::max(1, sharing)) * per;
    for (int i = 0; i < per && first + i < static_cast<int>(all.size()); ++i) hc.attn.push_back(all[first + i]);
    hc.pinned = true;
    return hc;
}

void pin_thread(const std::vector<int>& cores) {
    if (cores.empty()) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : cores) CPU_SET(c, &set);
    pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
}

void host_gqa_decode(const uint16_t* q, const uint16_t* kc, const uint16_t* vc, const int32_t* ctx, int T,
                     int nq, int nkv, int max_ctx, uint16_t* out, int threads) {
    const int G = nq / nkv;
    const float scale = 1.0f / std::sqrt(static_cast<float>(kD));
    const int ldsc = host_gqa_ldsc(max_ctx);
    if (threads <= 0) threads = omp_get_num_procs();
#pragma omp parallel num_threads(threads)
    {
        std::vector<float> sc(host_gqa_scratch_floats(max_ctx));
#pragma omp for collapse(2) schedule(dynamic, 1)
        for (int t = 0; t < T; ++t)
            for (int h = 0; h < nkv; ++h) {
                const size_t base = (static_cast<size_t>(t) * nkv + h) * max_ctx * kD;
                const size_t qo = (static_cast<size_t>(t) * nq + h * G) * kD;
                host_gqa_item(q + qo, kc + base, vc + base, ctx[t], G, scale, sc.data(), ldsc, out + qo);
            }
    }
}

}  // namespace mlt
