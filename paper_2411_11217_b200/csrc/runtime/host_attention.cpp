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

#pragma omp parallel num_threads(threads)
    {
        std::vector<float> sc(static_cast<size_t>(kMaxG) * max_ctx_);
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

                __m512 q[kMaxG][kD / 16];
                for (int g = 0; g < G; ++g)
                    for (int c = 0; c < kD / 16; ++c)
                        q[g][c] = _mm512_mul_ps(load_bf16x16(row + (h * G + g) * kD + c * 16), _mm512_set1_ps(scale));
                float mx[kMaxG];
                for (int g = 0; g < G; ++g) mx[g] = -INFINITY;
                for (int j = 0; j < L; ++j) {
                    __m512 k[kD / 16];
                    for (int c = 0; c < kD / 16; ++c) k[c] = load_bf16x16(kc + static_cast<size_t>(j) * kD + c * 16);
                    for (int g = 0; g < G; ++g) {
                        __m512 acc = _mm512_mul_ps(q[g][0], k[0]);
                        for (int c = 1; c < kD / 16; ++c) acc = _mm512_fmadd_ps(q[g][c], k[c], acc);
                        const float s = _mm512_reduce_add_ps(acc);
                        sc[static_cast<size_t>(g) * max_ctx_ + j] = s;
                        mx[g] = s > mx[g] ? s : mx[g];
                    }
                }
                __m512 o[kMaxG][kD / 16];
                float den[kMaxG];
                for (int g = 0; g < G; ++g) {
                    den[g] = 0.f;
                    for (int c = 0; c < kD / 16; ++c) o[g][c] = _mm512_setzero_ps();
                    float* s = sc.data() + static_cast<size_t>(g) * max_ctx_;
                    for (int j = 0; j < L; ++j) {
                        s[j] = std::exp(s[j] - mx[g]);
                        den[g] += s[j];
                    }
                }
                for (int j = 0; j < L; ++j) {
                    __m512 v[kD / 16];
                    for (int c = 0; c < kD / 16; ++c) v[c] = load_bf16x16(vc + static_cast<size_t>(j) * kD + c * 16);
                    for (int g = 0; g < G; ++g) {
                        const __m512 pj = _mm512_set1_ps(sc[static_cast<size_t>(g) * max_ctx_ + j]);
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
