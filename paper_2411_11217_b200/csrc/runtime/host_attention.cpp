// Host-core GQA decode attention — the paper's default placement (A_g = 0,
// PAPER.md:390-392 "CPU attention = the softmax part", 553 "customized CPU
// GQA kernels").  It is a policy choice, not a fallback: the task is
// TaskKind::CpuAttn on Resource::Cpu of the CGOPipe DAG.
//
// Input: the D1 offload of one micro-batch (bf16 rows q|k|v, roped).  The
// new k/v are appended to the host KV cache, laid out head-major
// [layer][seq][kv_head][ctx][d] so each (seq, head) is one contiguous stream
// for the hardware prefetcher.  One work item per (seq, kv head) computes all
// G = n_q/n_kv query heads against one pass over K and V (GQA reuse), in
// fp32 with AVX-512 (bf16 -> fp32 by shift).  Output is written straight in
// the packed operand layout of the O projection, so the D2 upload needs no
// device-side repack.
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../kernels/common.cuh"
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

}  // namespace

void Runtime::host_attention(int l, int mb, int step) {
    const int G = nq_ / nkv_;
    const int t0 = mb * mu_;
    const uint16_t* qkv = h_qkv_ + static_cast<size_t>(mb) * mu_ * W_;
    uint8_t* out = h_attn_ + static_cast<size_t>(mb) * Rmu_ * Ho_ * 2;  // this rank's heads
    const int32_t* pos = step_pos_.data() + static_cast<size_t>(step - 1) * N_;
    const float scale = 1.0f / std::sqrt(static_cast<float>(kD));
    // Default: all cores but two, which stay free for the resource launcher
    // threads (a descheduled GPU launcher leaves the device idle between
    // kernels of one PostAttn).
    // Under TP every rank's process shares the node's host cores; a
    // shard-only measurement runs one rank alone on its slice of the node.
    const int sharing = opt_.tp_shard_only ? 1 : shard_.size;
    const int threads = opt_.host_threads > 0 ? opt_.host_threads
                                              : std::max(1, (omp_get_num_procs() - 2) / sharing);

    // AVX512-BF16 dot products when the host has them (SPR+); otherwise the
    // fp32 FMA path.  Score rows are padded to whole 16-key blocks.
    static const bool bf16dot = __builtin_cpu_supports("avx512bf16");
    const int ldsc = (max_ctx_ + 15) & ~15;
#pragma omp parallel num_threads(threads)
    {
        std::vector<float> sc(static_cast<size_t>(kMaxG) * ldsc);
#pragma omp for collapse(2) schedule(dynamic, 1)
        for (int t = 0; t < mu_; ++t)
            for (int h = 0; h < nkv_; ++h) {
                const int seq = t0 + t;
                const int p = pos[seq];
                const int L = p + 1;
                const uint16_t* row = qkv + static_cast<size_t>(t) * W_;
                const size_t base = ((static_cast<size_t>(l) * N_ + seq) * nkv_ + h) * max_ctx_;
                uint16_t* kc = h_kcache_ + base * kD;
                uint16_t* vc = h_vcache_ + base * kD;
                std::memcpy(kc + static_cast<size_t>(p) * kD, row + (nq_ + h) * kD, kD * 2);
                std::memcpy(vc + static_cast<size_t>(p) * kD, row + (nq_ + nkv_ + h) * kD, kD * 2);

                float mx[kMaxG];
                for (int g = 0; g < G; ++g) mx[g] = -INFINITY;
                if (bf16dot) {
                    // 16 keys per pass: 4 VDPBF16PS per key (q and k stay bf16,
                    // fp32 accumulate), one transpose-add tree per 16 keys
                    for (int g = 0; g < G; ++g) {
                        __m512bh qb[4];
                        const uint16_t* qr = row + (h * G + g) * kD;
                        for (int c = 0; c < 4; ++c) qb[c] = (__m512bh)_mm512_loadu_si512(qr + 32 * c);
                        float* srow = sc.data() + static_cast<size_t>(g) * ldsc;
                        __m512 m16 = _mm512_set1_ps(-INFINITY);
                        for (int j0 = 0; j0 < L; j0 += 16) {
                            const int n = std::min(16, L - j0);
                            const __mmask16 live = static_cast<__mmask16>((1u << n) - 1u);
                            const __m512 s16 = _mm512_mask_mov_ps(
                                _mm512_set1_ps(-INFINITY), live,
                                _mm512_mul_ps(scores16_bf16(qb, kc + static_cast<size_t>(j0) * kD, n),
                                              _mm512_set1_ps(scale)));
                            _mm512_storeu_ps(srow + j0, s16);
                            m16 = _mm512_max_ps(m16, s16);
                        }
                        mx[g] = _mm512_reduce_max_ps(m16);
                    }
                } else {
                    __m512 q[kMaxG][kD / 16];
                    for (int g = 0; g < G; ++g)
                        for (int c = 0; c < kD / 16; ++c)
                            q[g][c] = _mm512_mul_ps(load_bf16x16(row + (h * G + g) * kD + c * 16), _mm512_set1_ps(scale));
                    for (int j = 0; j < L; ++j) {
                        __m512 k[kD / 16];
                        for (int c = 0; c < kD / 16; ++c) k[c] = load_bf16x16(kc + static_cast<size_t>(j) * kD + c * 16);
                        for (int g = 0; g < G; ++g) {
                            __m512 acc = _mm512_mul_ps(q[g][0], k[0]);
                            for (int c = 1; c < kD / 16; ++c) acc = _mm512_fmadd_ps(q[g][c], k[c], acc);
                            const float s = _mm512_reduce_add_ps(acc);
                            sc[static_cast<size_t>(g) * ldsc + j] = s;
                            mx[g] = s > mx[g] ? s : mx[g];
                        }
                    }
                    for (int g = 0; g < G; ++g)  // pad the tail block like the bf16 path
                        for (int j = L; j < ((L + 15) & ~15); ++j) sc[static_cast<size_t>(g) * ldsc + j] = -INFINITY;
                }
                __m512 o[kMaxG][kD / 16];
                float den[kMaxG];
                for (int g = 0; g < G; ++g) {  // vectorised softmax numerators (tail lanes -> 0)
                    for (int c = 0; c < kD / 16; ++c) o[g][c] = _mm512_setzero_ps();
                    float* srow = sc.data() + static_cast<size_t>(g) * ldsc;
                    const __m512 m = _mm512_set1_ps(mx[g]);
                    __m512 d16 = _mm512_setzero_ps();
                    for (int j0 = 0; j0 < L; j0 += 16) {
                        const int n = std::min(16, L - j0);
                        const __mmask16 live = static_cast<__mmask16>((1u << n) - 1u);
                        const __m512 e = _mm512_maskz_mov_ps(live, exp16(_mm512_sub_ps(_mm512_loadu_ps(srow + j0), m)));
                        _mm512_storeu_ps(srow + j0, e);
                        d16 = _mm512_add_ps(d16, e);
                    }
                    den[g] = _mm512_reduce_add_ps(d16);
                }
                for (int j = 0; j < L; ++j) {
                    __m512 v[kD / 16];
                    for (int c = 0; c < kD / 16; ++c) v[c] = load_bf16x16(vc + static_cast<size_t>(j) * kD + c * 16);
                    for (int g = 0; g < G; ++g) {
                        const __m512 pj = _mm512_set1_ps(sc[static_cast<size_t>(g) * ldsc + j]);
                        for (int c = 0; c < kD / 16; ++c) o[g][c] = _mm512_fmadd_ps(pj, v[c], o[g][c]);
                    }
                }
                for (int g = 0; g < G; ++g) {
                    const __m512 inv = _mm512_set1_ps(1.0f / den[g]);
                    alignas(64) float buf[kD];
                    for (int c = 0; c < kD / 16; ++c) _mm512_store_ps(buf + c * 16, _mm512_mul_ps(o[g][c], inv));
                    alignas(16) uint16_t ob[kD];
                    for (int i = 0; i < kD; ++i) ob[i] = f32_to_bf16(buf[i]);
                    const int col = (h * G + g) * kD;
                    for (int i = 0; i < kD; i += 8)
                        std::memcpy(out + mltk::b_packed_off(t, col + i, Rmu_), ob + i, 16);
                }
            }
    }
}

}  // namespace mlt
