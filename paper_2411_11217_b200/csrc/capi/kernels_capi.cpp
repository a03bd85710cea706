// C ABI over the sm_100a kernels (include/mlt.h, "Kernel-level entry
// points").  Thin: argument checks, cudaError -> MLT_ERR_CUDA, no hidden
// allocation except mlt_expert_ffn's (none: all buffers caller-owned).
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "../kernels/kernels.hpp"
#include "../runtime/host_layout.hpp"
#include "../runtime/host_gqa.hpp"
#include "../runtime/weight_codec.hpp"

#include <algorithm>
#include <functional>
#include <vector>
#include "lightplan/pipesim.hpp"
#include "lightplan/planner.hpp"
#include "lightplan/batcher.hpp"
#include "status.hpp"

namespace {

template <class F>
int guard(F&& f) {
    MLT_GUARD_BODY(lightplan)
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw mlt::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// SM count of the calling thread's current device (cached per device)
int sm_count() {
    static std::atomic<int> cache[64] = {};
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev >= 0 && dev < 64 && cache[dev].load()) return cache[dev].load();
    int n = 0;
    ck(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
    if (dev >= 0 && dev < 64) cache[dev].store(n);
    return n;
}

cudaStream_t st(void* s) { return reinterpret_cast<cudaStream_t>(s); }

mltk::GemmArgs to_args(const mlt_gemm_args_t* a) {
    mltk::GemmArgs g;
    g.a_table = reinterpret_cast<const uint8_t* const*>(a->a_table);
    g.n_mats = a->n_mats;
    g.G = a->G;
    g.RB = a->RB;
    g.K = a->K;
    g.b = reinterpret_cast<const uint8_t*>(a->b);
    g.R = a->R;
    g.b_off = a->b_off;
    g.b_cnt = a->b_cnt;
    g.rows_dense = a->rows_dense;
    g.n_cap = a->n_cap;
    g.epi = a->epi;
    g.alpha = a->alpha;
    g.out_f32 = a->out_f32;
    g.ldo = a->ldo;
    g.residual = a->residual;
    g.ldr = a->ldr;
    g.out_packed = reinterpret_cast<uint8_t*>(a->out_packed);
    g.out_R = a->out_R;
    g.n_chunks = a->n_chunks > 0 ? a->n_chunks : 1;
    g.k_splits = a->k_splits > 0 ? a->k_splits : 1;
    g.split_stride = a->split_stride;
    g.trace = a->trace;
    g.codec = a->codec;
    g.ktrace = a->ktrace;
    g.sk_scratch = a->sk_scratch;
    g.sk_count = reinterpret_cast<unsigned long long*>(a->sk_count);
    g.sk_rows = a->sk_rows;
    if (a->dec_groups > 0) g.dec_groups = a->dec_groups;
    g.codec_raw = a->codec_raw;
    g.enc_tile = a->enc_tile;
    return g;
}

}  // namespace

extern "C" {

int mlt_pack_weight(const uint16_t* src, int64_t M, int64_t K, uint16_t* dst) {
    return guard([&] {
        if (M % 128 || K % 64 || M <= 0 || K <= 0) throw std::invalid_argument("pack_weight: M%128, K%64");
        mlt::pack_weight(src, M, K, dst);
        return MLT_OK;
    });
}

int mlt_codec_encode(const uint8_t* packed, int64_t M, int64_t K, uint8_t* out) {
    return guard([&] {
        if (M % 128 || K % 64 || M <= 0 || K <= 0) throw std::invalid_argument("codec_encode: M%128, K%64");
        const int64_t tiles = M / 128 * (K / 64);
        int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
        for (int64_t t = 0; t < tiles; ++t)
            bad += mlt::codec_encode_tile(packed + t * 16384, out + t * mlt::kCodecTileBytes) ? 0 : 1;
        if (bad) throw std::invalid_argument("codec_encode: " + std::to_string(bad) + " tile(s) need > " +
                                             std::to_string(mlt::kCodecMaxEscapes) + " escapes");
        return MLT_OK;
    });
}

int mlt_codec_decode(const uint8_t* enc, int64_t tiles, uint8_t* packed) {
    return guard([&] {
        for (int64_t t = 0; t < tiles; ++t)
            mlt::codec_decode_tile(enc + t * mlt::kCodecTileBytes, packed + t * 16384);
        return MLT_OK;
    });
}

int mlt_codec_tile_bytes(void) { return mlt::kCodecTileBytes; }

// Encode an [M, K] packed matrix in a reordered code (fragment / row-plane
// order) with the per-block raw fallback: a 128-row block with a tile the
// code cannot hold is stored as 16 KiB raw tiles (raw_tile: packed -> the
// engine's raw layout), its flag set in raw_blocks; without raw_blocks such
// a block is an error.  Returns the number of raw blocks.
static int encode_blocks(const char* what, const uint8_t* packed, int64_t M, int64_t K, uint8_t* out,
                         uint8_t* raw_blocks, const std::function<bool(const uint8_t*, uint8_t*)>& enc,
                         void (*raw_tile)(const uint8_t*, uint8_t*), int tile_bytes = mlt::kCodecTileBytes,
                         int max_escapes = mlt::kCodecMaxEscapes) {
    if (M % 128 || K % 64 || M <= 0 || K <= 0) throw std::invalid_argument(std::string(what) + ": M%128, K%64");
    const int64_t kb = K / 64, rbs = M / 128;
    std::vector<int64_t> off(rbs + 1, 0);
    std::vector<uint8_t> raw(rbs, 0);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t r = 0; r < rbs; ++r) {
        std::vector<uint8_t> tmp_v(std::max(mlt::kCodecTileBytes, mlt::codec4_tile_bytes(mlt::kCodec4CapLimit)));
        uint8_t* tmp = tmp_v.data();
        for (int64_t t = 0; t < kb; ++t)
            if (!enc(packed + (r * kb + t) * 16384, tmp)) {
                raw[r] = 1;
                ++bad;
                break;
            }
    }
    if (bad && !raw_blocks)
        throw std::invalid_argument(std::string(what) + ": " + std::to_string(bad) + " row block(s) need > " +
                                    std::to_string(max_escapes) + " escapes in a tile");
    for (int64_t r = 0; r < rbs; ++r) off[r + 1] = off[r] + kb * (raw[r] ? 16384 : tile_bytes);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rbs; ++r)
        for (int64_t t = 0; t < kb; ++t) {
            const uint8_t* src = packed + (r * kb + t) * 16384;
            if (raw[r])
                raw_tile(src, out + off[r] + t * 16384);
            else
                enc(src, out + off[r] + t * tile_bytes);
        }
    if (raw_blocks) std::memcpy(raw_blocks, raw.data(), static_cast<size_t>(rbs));
    return bad;
}

int mlt_codec_encode_frag(const uint8_t* packed, int64_t M, int64_t K, uint8_t* out, uint8_t* raw_blocks) {
    return guard([&] {
        return encode_blocks("codec_encode_frag", packed, M, K, out, raw_blocks, mlt::codec_encode_frag_tile,
                             [](const uint8_t* src, uint8_t* dst) {
                                 mlt::frag_from_packed(src, reinterpret_cast<uint16_t*>(dst));
                             });
    });
}

int mlt_codec_encode_rows(const uint8_t* packed, int64_t M, int64_t K, uint8_t* out, uint8_t* raw_blocks) {
    return guard([&] {
        return encode_blocks("codec_encode_rows", packed, M, K, out, raw_blocks, mlt::codec_encode_rows_tile,
                             [](const uint8_t* src, uint8_t* dst) { std::memcpy(dst, src, 16384); });
    });
}

int mlt_codec4_encode_rows_cap(const uint8_t* packed, int64_t M, int64_t K, int32_t cap, uint8_t* out,
                               uint8_t* raw_blocks) {
    return guard([&] {
        if (cap < 0 || cap > mlt::kCodec4CapLimit) throw std::invalid_argument("codec4_encode_rows: cap in [0, 200]");
        return encode_blocks("codec4_encode_rows", packed, M, K, out, raw_blocks,
                             [cap](const uint8_t* a, uint8_t* b) { return mlt::codec4_encode_rows_tile(a, b, cap); },
                             [](const uint8_t* src, uint8_t* dst) { std::memcpy(dst, src, 16384); },
                             mlt::codec4_tile_bytes(cap), cap);
    });
}

int mlt_codec4_encode_rows(const uint8_t* packed, int64_t M, int64_t K, uint8_t* out, uint8_t* raw_blocks) {
    return mlt_codec4_encode_rows_cap(packed, M, K, mlt::kCodec4MaxEntries, out, raw_blocks);
}

int mlt_codec4_decode_rows_cap(const uint8_t* enc, int64_t tiles, int32_t cap, uint8_t* packed) {
    return guard([&] {
        if (cap < 0 || cap > mlt::kCodec4CapLimit) throw std::invalid_argument("codec4_decode_rows: cap in [0, 200]");
        const int tb = mlt::codec4_tile_bytes(cap);
        for (int64_t t = 0; t < tiles; ++t) mlt::codec4_decode_rows_tile(enc + t * tb, packed + t * 16384);
        return MLT_OK;
    });
}

int mlt_codec4_decode_rows(const uint8_t* enc, int64_t tiles, uint8_t* packed) {
    return mlt_codec4_decode_rows_cap(enc, tiles, mlt::kCodec4MaxEntries, packed);
}

int mlt_codec4_tile_bytes(void) { return mlt::kCodec4TileBytes; }
int mlt_codec4_tile_bytes_for(int32_t cap) { return mlt::codec4_tile_bytes(cap); }

int mlt_frag_pack(const uint8_t* packed, int64_t tiles, uint8_t* out) {
    return guard([&] {
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < tiles; ++t)
            mlt::frag_from_packed(packed + t * 16384, reinterpret_cast<uint16_t*>(out + t * 16384));
        return MLT_OK;
    });
}

int mlt_host_gqa_use_amx(int enable) { return mlt::host_gqa_set_amx(enable != 0) ? 1 : 0; }

int mlt_host_gqa_decode(const uint16_t* q, const uint16_t* kc, const uint16_t* vc, const int32_t* ctx, int T,
                        int nq, int nkv, int d, int max_ctx, uint16_t* out, int threads) {
    return guard([&] {
        if (d != 128 || nkv <= 0 || nq % nkv || nq / nkv > 16 || T < 0 || max_ctx <= 0)
            throw std::invalid_argument("host_gqa_decode: d == 128, nq % nkv == 0, nq / nkv <= 16");
        for (int t = 0; t < T; ++t)
            if (ctx[t] < 1 || ctx[t] > max_ctx) throw std::invalid_argument("host_gqa_decode: 1 <= ctx[t] <= max_ctx");
        mlt::host_gqa_decode(q, kc, vc, ctx, T, nq, nkv, max_ctx, out, threads);
        return MLT_OK;
    });
}

int mlt_unpack_rows(const uint8_t* packed, int64_t R, int64_t rows, int64_t K, uint16_t* dst) {
    return guard([&] {
        if (K % 64 || R % 8 || rows > R) throw std::invalid_argument("unpack_rows: K%64, R%8, rows<=R");
        mlt::unpack_rows(packed, R, rows, K, dst);
        return MLT_OK;
    });
}

int mlt_pack_rows_host(const uint16_t* src, int64_t rows, int64_t K, int64_t R, uint8_t* dst) {
    return guard([&] {
        if (K % 64 || R % 8 || rows > R) throw std::invalid_argument("pack_rows: K%64, R%8, rows<=R");
        mlt::pack_rows(src, rows, K, R, dst);
        return MLT_OK;
    });
}

int mlt_gemm(const mlt_gemm_args_t* a, void* stream) {
    return guard([&] {
        ck(mltk::launch_gemm(to_args(a), sm_count(), st(stream)), "gemm");
        return MLT_OK;
    });
}

int mlt_embed(const int32_t* tokens, const uint16_t* table, int T, int H, float* x, void* s) {
    return guard([&] {
        ck(mltk::launch_embed(tokens, table, T, H, x, st(s)), "embed");
        return MLT_OK;
    });
}

int mlt_rmsnorm_pack(const float* x, const uint16_t* gamma, int T, int H, float eps, void* out,
                     int R, void* s) {
    return guard([&] {
        ck(mltk::launch_rmsnorm_pack(x, gamma, T, H, eps, reinterpret_cast<uint8_t*>(out), R, st(s)),
           "rmsnorm_pack");
        return MLT_OK;
    });
}

int mlt_pack_rows(const uint16_t* src, int ld, int T, int K, void* dst, int R, void* s) {
    return guard([&] {
        ck(mltk::launch_pack_rows(src, ld, T, K, reinterpret_cast<uint8_t*>(dst), R, st(s)), "pack_rows");
        return MLT_OK;
    });
}

int mlt_rope_qkv(const float* qkv, const int32_t* pos, const void* rope, int T, int nq, int nkv,
                 int d, uint16_t* out, void* s) {
    return guard([&] {
        ck(mltk::launch_rope_qkv(qkv, 1, 0, pos, reinterpret_cast<const float2*>(rope), T, nq, nkv, d, out,
                                 st(s)),
           "rope_qkv");
        return MLT_OK;
    });
}

int mlt_router_topk(const float* x, const uint16_t* gamma, float eps, const uint16_t* hn_in,
                    const uint16_t* w, int T, int H, int E, int K, uint16_t* hn_out, float* logits,
                    int32_t* idx, float* wts, void* s) {
    return guard([&] {
        ck(mltk::launch_router(x, gamma, eps, hn_in, w, T, H, E, K, hn_out, logits, idx, wts, st(s)),
           "router");
        return MLT_OK;
    });
}

int mlt_moe_permute(const int32_t* idx, const uint16_t* hn, int T, int H, int E, int K,
                    int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv, void* xp, int R,
                    void* s) {
    return guard([&] {
        ck(mltk::launch_moe_permute(idx, hn, T, H, E, K, counts, offsets, perm, inv,
                                    reinterpret_cast<uint8_t*>(xp), R, st(s)),
           "moe_permute");
        return MLT_OK;
    });
}

int mlt_moe_combine(const float* h, const float* y, int ldy, const int32_t* inv, const float* w,
                    int T, int H, int K, float* x, void* s) {
    return guard([&] {
        ck(mltk::launch_moe_combine(h, y, ldy, inv, w, T, H, K, x, st(s)), "moe_combine");
        return MLT_OK;
    });
}

int mlt_expert_ffn(const void* xp, int R, const int32_t* counts, const int32_t* offsets,
                   const void* w13, const void* w2, int E, int H, int F, int n_cap, void* inter,
                   float* y, const int32_t* inv, const float* wts, const float* h, int T, int K,
                   float* x_out, void* s) {
    return guard([&] {
        if (H % 128 || F % 128) throw std::invalid_argument("expert_ffn: H, F must be multiples of 128");
        mltk::GemmArgs g;
        g.a_table = reinterpret_cast<const uint8_t* const*>(w13);
        g.n_mats = 2;
        g.G = E;
        g.RB = F / 128;
        g.K = H;
        g.b = reinterpret_cast<const uint8_t*>(xp);
        g.R = R;
        g.b_off = offsets;
        g.b_cnt = counts;
        g.n_cap = n_cap;
        g.epi = mltk::kEpiSiluPacked;
        g.out_packed = reinterpret_cast<uint8_t*>(inter);
        g.out_R = R;
        ck(mltk::launch_gemm(g, sm_count(), st(s)), "expert gate/up");
        mltk::GemmArgs d;
        d.a_table = reinterpret_cast<const uint8_t* const*>(w2);
        d.n_mats = 1;
        d.G = E;
        d.RB = H / 128;
        d.K = F;
        d.b = reinterpret_cast<const uint8_t*>(inter);
        d.R = R;
        d.b_off = offsets;
        d.b_cnt = counts;
        d.n_cap = n_cap;
        d.epi = mltk::kEpiF32;
        d.out_f32 = y;
        d.ldo = H;
        ck(mltk::launch_gemm(d, sm_count(), st(s)), "expert down");
        if (x_out) ck(mltk::launch_moe_combine(h, y, H, inv, wts, T, H, K, x_out, st(s)), "combine");
        return MLT_OK;
    });
}

int mlt_argmax(const float* logits, int T, int V, int32_t* ids, float* margin, void* s) {
    return guard([&] {
        ck(mltk::launch_argmax(logits, T, V, ids, margin, st(s)), "argmax");
        return MLT_OK;
    });
}

int mlt_gqa_decode_paged(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp,
                         const int32_t* bt, int max_pages, const int32_t* seq, const int32_t* ctx,
                         int T, int nq, int nkv, int d, int page, void* out_packed, int R,
                         float* out_f, void* s) {
    return guard([&] {
        ck(mltk::launch_gqa_decode_paged(q, ldq, kp, vp, bt, max_pages, seq, ctx, T, nq, nkv, d, page,
                                         reinterpret_cast<uint8_t*>(out_packed), R, out_f, st(s)),
           "gqa_decode_paged");
        return MLT_OK;
    });
}

int mlt_gqa_decode_paged_split(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp,
                               const int32_t* bt, int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                               int nq, int nkv, int d, int page, void* out_packed, int R, float* out_f,
                               int splits, int max_splits, float* scratch, int32_t* counters, void* s) {
    return guard([&] {
        if (splits < 0 || max_splits < 1 || !scratch || !counters)
            throw std::invalid_argument("gqa_decode_paged_split: splits >= 0, max_splits >= 1, scratch + counters");
        mltk::GqaSplit sp;
        sp.splits = splits;
        sp.max_splits = max_splits;
        sp.scratch = scratch;
        sp.counters = counters;
        ck(mltk::launch_gqa_decode_paged(q, ldq, kp, vp, bt, max_pages, seq, ctx, T, nq, nkv, d, page,
                                         reinterpret_cast<uint8_t*>(out_packed), R, out_f, st(s), &sp),
           "gqa_decode_paged_split");
        return MLT_OK;
    });
}

int mlt_gqa_decode_paged_flat(const uint16_t* q, int ldq, const uint16_t* kp, const uint16_t* vp, const int32_t* bt,
                              int max_pages, const int32_t* seq, const int32_t* ctx, int T, int nq, int nkv, int d,
                              int page, void* out_packed, int R, float* out_f, int ctas, float* scratch,
                              int32_t* counters, void* s) {
    return guard([&] {
        mltk::GqaFlat fl;
        fl.ctas = ctas > 0 ? ctas : mltk::gqa_flat_ctas(sm_count());
        fl.scratch = scratch;
        fl.counters = counters;
        ck(mltk::launch_gqa_decode_flat(q, ldq, kp, vp, bt, max_pages, seq, ctx, T, nq, nkv, d, page,
                                        reinterpret_cast<uint8_t*>(out_packed), R, out_f, fl, st(s)),
           "gqa_decode_paged_flat");
        return MLT_OK;
    });
}

int mlt_kv_append(const uint16_t* qkv, int nq, int nkv, int d, const int32_t* seq,
                  const int32_t* pos, int T, const int32_t* bt, int max_pages, int page,
                  uint16_t* kp, uint16_t* vp, void* s) {
    return guard([&] {
        ck(mltk::launch_kv_append(qkv, nq, nkv, d, seq, pos, T, bt, max_pages, page, kp, vp, st(s)),
           "kv_append");
        return MLT_OK;
    });
}

int mlt_prefill_attention(const uint16_t* qkv, int W, const int32_t* tiles, int n_tiles, int nq, int nkv,
                          int d, void* out_packed, int R, void* s) {
    return guard([&] {
        ck(mltk::launch_prefill_attention(qkv, W, reinterpret_cast<const int4*>(tiles), n_tiles, nq, nkv, d,
                                          reinterpret_cast<uint8_t*>(out_packed), R, st(s)),
           "prefill_attention");
        return MLT_OK;
    });
}

int mlt_kv_stage(const uint16_t* qkv, int W, int nq, int nkv, int d, const int32_t* tok_seq,
                 const int32_t* tok_pos, const int32_t* seq_row0, const int32_t* seq_len, int T,
                 uint16_t* stage_k, uint16_t* stage_v, void* s) {
    return guard([&] {
        ck(mltk::launch_kv_stage(qkv, W, nq, nkv, d, tok_seq, tok_pos, seq_row0, seq_len, T, stage_k, stage_v,
                                 st(s)),
           "kv_stage");
        return MLT_OK;
    });
}

int mlt_rope_table(int max_pos, int d, double theta, float* out) {
    return guard([&] {
        const int half = d / 2;
        for (int p = 0; p < max_pos; ++p)
            for (int i = 0; i < half; ++i) {
                const double inv = std::pow(theta, -2.0 * static_cast<double>(i) / static_cast<double>(d));
                const double ang = static_cast<double>(p) * inv;
                out[(static_cast<int64_t>(p) * half + i) * 2] = static_cast<float>(std::cos(ang));
                out[(static_cast<int64_t>(p) * half + i) * 2 + 1] = static_cast<float>(std::sin(ang));
            }
        return MLT_OK;
    });
}

int mlt_measure_link(int device, size_t bytes, int reps, double out[3]) {
    return guard([&] {
        ck(cudaSetDevice(device), "set device");
        const size_t align = 2u << 20;
        bytes = (bytes + align - 1) / align * align;
        void* h = std::aligned_alloc(align, bytes);
        if (!h) throw std::bad_alloc();
        std::memset(h, 1, bytes);
        void* h2 = nullptr;
        void* d = nullptr;
        void* d2 = nullptr;
        cudaStream_t s1 = nullptr, s2 = nullptr;
        cudaEvent_t a, b;
        auto cleanup = [&] {
            if (d) cudaFree(d);
            if (d2) cudaFree(d2);
            if (h2) cudaFreeHost(h2);
            cudaHostUnregister(h);
            std::free(h);
            if (s1) cudaStreamDestroy(s1);
            if (s2) cudaStreamDestroy(s2);
        };
        try {
            ck(cudaHostRegister(h, bytes, cudaHostRegisterDefault), "register");
            ck(cudaMalloc(&d, bytes), "malloc");
            ck(cudaMalloc(&d2, 64u << 20), "malloc");
            ck(cudaHostAlloc(&h2, 64u << 20, 0), "hostalloc");
            ck(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking), "stream");
            ck(cudaEventCreate(&a), "event");
            ck(cudaEventCreate(&b), "event");
            auto best = [&](cudaMemcpyKind kind, bool concurrent) {
                double bw = 0;
                for (int r = 0; r < reps; ++r) {
                    ck(cudaEventRecord(a, s1), "record");
                    if (kind == cudaMemcpyHostToDevice) ck(cudaMemcpyAsync(d, h, bytes, kind, s1), "copy");
                    else ck(cudaMemcpyAsync(h, d, bytes, kind, s1), "copy");
                    if (concurrent)
                        for (int i = 0; i < 8; ++i) ck(cudaMemcpyAsync(h2, d2, 1u << 20, cudaMemcpyDeviceToHost, s2), "copy");
                    ck(cudaEventRecord(b, s1), "record");
                    ck(cudaEventSynchronize(b), "sync");
                    ck(cudaStreamSynchronize(s2), "sync");
                    float ms = 0;
                    ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
                    bw = std::max(bw, static_cast<double>(bytes) / (ms * 1e-3) / 1e9);
                }
                return bw;
            };
            best(cudaMemcpyHostToDevice, false);  // warm
            out[0] = best(cudaMemcpyHostToDevice, false);
            out[1] = best(cudaMemcpyDeviceToHost, false);
            out[2] = best(cudaMemcpyHostToDevice, true);
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
        return MLT_OK;
    });
}

// Read: 64-byte vector loads into four independent accumulators per thread
// (a scalar `sum += a[i]` chain is add-latency bound, not DRAM bound, and
// under-reports the host by ~2x); copy: plain vectorised loop.  Pages are
// first-touched by the threads that read them.
int mlt_measure_host_bw(size_t bytes, double out[2]) {
    return guard([&] {
        const size_t n = bytes / 64 * 16;  // floats, whole 64-byte lines
        float* a = static_cast<float*>(std::aligned_alloc(64, n * 4));
        float* b = static_cast<float*>(std::aligned_alloc(64, n * 4));
        if (!a || !b) {
            std::free(a);
            std::free(b);
            throw std::runtime_error("measure_host_bw: allocation failed");
        }
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) a[i] = 1.0f, b[i] = 0.0f;
        double best_read = 0, best_copy = 0;
        for (int rep = 0; rep < 3; ++rep) {
            float sum = 0;
            auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for reduction(+ : sum) schedule(static)
            for (int64_t i = 0; i < static_cast<int64_t>(n); i += 64) {
                __m512 s0 = _mm512_load_ps(a + i), s1 = _mm512_load_ps(a + i + 16);
                s0 = _mm512_add_ps(s0, _mm512_load_ps(a + i + 32));
                s1 = _mm512_add_ps(s1, _mm512_load_ps(a + i + 48));
                sum += _mm512_reduce_add_ps(_mm512_add_ps(s0, s1));
            }
            auto t1 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < static_cast<int64_t>(n); i += 16) _mm512_store_ps(b + i, _mm512_load_ps(a + i));
            auto t2 = std::chrono::steady_clock::now();
            if (sum < 0) throw std::runtime_error("unreachable");
            best_read = std::max(best_read, n * 4.0 / std::chrono::duration<double>(t1 - t0).count() / 1e9);
            best_copy = std::max(best_copy, n * 8.0 / std::chrono::duration<double>(t2 - t1).count() / 1e9);
        }
        std::free(a);
        std::free(b);
        out[0] = best_read;
        out[1] = best_copy;
        return MLT_OK;
    });
}

int mlt_synth_bf16(uint64_t seed, uint64_t tid, int64_t n, float scale, int is_norm, uint16_t* out) {
    return guard([&] {
        mlt::synth_bf16(seed, tid, 0, n, scale, is_norm != 0, out);
        return MLT_OK;
    });
}

}  // extern "C"
