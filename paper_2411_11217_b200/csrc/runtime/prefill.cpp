// GPU prefill stage.
//
// "we adopt the zigzag computation order proposed in FlexGen:
// loading the weights from CPU and performing the computation layer by
// layer.  For the prefill stage, we perform all the computation on GPU and
// offload KV cache to CPU for all the micro-batches."  The reference models
// it as layers * max(weight stream, prompt compute) (planner.cpp:110-150).
//
// B200 mapping.  Layer l's streamed weights go into pool slot (l+1)&1 over a
// dedicated copy stream while layer l-1 computes (the same two-slot pool and
// page tables the decode uses).  Prompt tokens are processed in chunks of
// whole sequences (capacity pf_T_ tokens, sized from the budget left in the
// arena); between layers the fp32 residual of every prompt token lives in a
// page-locked host store, so a chunk's residual is uploaded on the H2D
// stream, computed, and written back on the D2H stream with its K/V rows —
// double-buffered, so both copies overlap the neighbouring chunk's compute.
// Per chunk the kernels are the decode's (RMSNorm-pack, paged swap-AB
// tcgen05 GEMMs, rope, router, permute, expert GEMMs, combine) at T rows,
// plus the causal prefill attention (attention_prefill.cu).
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kernels/kernels.hpp"
#include "host_layout.hpp"
#include "runtime.hpp"
#include "runtime_util.hpp"

namespace mlt {

using detail::ck;
using detail::host_alloc;
using detail::host_free;
using detail::round_up;

namespace {

constexpr int kMetaPerToken = 15;  // int32 metadata entries per token of chunk capacity

struct Chunk {
    int seq0 = 0, n_seq = 0;   // sequences [seq0, seq0 + n_seq)
    int64_t tok0 = 0;          // first token (global, concatenated order)
    int tokens = 0;
    int n_tiles = 0;
};

}  // namespace

void Runtime::prefill_alloc(int64_t total_tokens, int max_len) {
    if (!pf_T_) {
        Arena& A = *arena_;
        const size_t Hs = static_cast<size_t>(H_), Ws = static_cast<size_t>(W_), Fs = static_cast<size_t>(F_);
        auto bytes_for = [&](size_t T) {
            const size_t R = static_cast<size_t>(round_up(static_cast<int>(T), 16));
            const size_t Re = static_cast<size_t>(round_up(static_cast<int>(T) * K_ + 16 * E_, 16));
            size_t b = 2 * T * Hs * 4 + R * std::max(Hs, static_cast<size_t>(Ho_)) * 2 + T * Ws * 2 + T * Hs * 4 +
                       T * Hs * 2 + T * K_ * 12 + Re * 4 + Re * Hs * 2 + Re * Fs * 2 +
                       std::max(Re * Hs * 4, R * Ws * 4) + 2 * static_cast<size_t>(kMetaPerToken) * T * 4;
            if (!policy_.attn_on_gpu) b += 2 * 2 * T * static_cast<size_t>(nkv_) * d_ * 2;
            return b + 16 * 1024;  // per-buffer alignment slack
        };
        const size_t free_b = A.capacity() - A.used();
        const size_t keep = 32u << 20;
        int T = std::min(16384 / K_, 8192);
        if (opt_.prefill_chunk_tokens > 0) T = std::min(T, round_up(opt_.prefill_chunk_tokens, 16));
        while (T > 16 && bytes_for(static_cast<size_t>(T)) + keep > free_b) T -= 16;
        if (T < max_len || bytes_for(static_cast<size_t>(T)) + keep > free_b)
            throw BudgetError("prefill: the budget leaves room for chunks of " + std::to_string(T) +
                              " tokens; the longest prompt has " + std::to_string(max_len));
        pf_T_ = T;
        pf_R_ = round_up(T, 16);
        pf_Re_ = round_up(T * K_ + 16 * E_, 16);
        const size_t Ts = static_cast<size_t>(T);
        for (int b = 0; b < 2; ++b) pf_x_[b] = static_cast<float*>(A.alloc(Ts * Hs * 4, "pf_x"));
        pf_xn_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(pf_R_) * std::max(Hs, static_cast<size_t>(Ho_)) * 2, "pf_xn"));
        pf_qkv_ = static_cast<uint16_t*>(A.alloc(Ts * Ws * 2, "pf_qkv"));
        pf_h_ = static_cast<float*>(A.alloc(Ts * Hs * 4, "pf_h"));
        pf_hn_ = static_cast<uint16_t*>(A.alloc(Ts * Hs * 2, "pf_hn"));
        pf_topk_ = static_cast<int32_t*>(A.alloc(Ts * K_ * 4, "pf_topk"));
        pf_topw_ = static_cast<float*>(A.alloc(Ts * K_ * 4, "pf_topw"));
        pf_inv_ = static_cast<int32_t*>(A.alloc(Ts * K_ * 4, "pf_inv"));
        pf_perm_ = static_cast<int32_t*>(A.alloc(static_cast<size_t>(pf_Re_) * 4, "pf_perm"));
        pf_xe_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(pf_Re_) * Hs * 2, "pf_xe"));
        pf_inter_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(pf_Re_) * Fs * 2, "pf_inter"));
        pf_y_ = static_cast<float*>(A.alloc(std::max(static_cast<size_t>(pf_Re_) * Hs, static_cast<size_t>(pf_R_) * Ws) * 4, "pf_y"));
        if (!policy_.attn_on_gpu)
            for (int b = 0; b < 2; ++b)
                pf_kst_[b] = static_cast<uint16_t*>(A.alloc(2 * Ts * nkv_ * d_ * 2, "pf_kv_stage"));
        pf_meta_cap_ = static_cast<int64_t>(kMetaPerToken) * T;
        pf_meta_ = static_cast<int32_t*>(A.alloc(2 * static_cast<size_t>(pf_meta_cap_) * 4, "pf_meta"));
    } else if (max_len > pf_T_) {
        throw BudgetError("prefill: prompt of " + std::to_string(max_len) + " tokens exceeds the chunk capacity " +
                          std::to_string(pf_T_) + " fixed by the first prefill");
    }
    if (total_tokens > h_pfx_tokens_) {
        host_free(h_pfx_, true);
        h_pfx_ = reinterpret_cast<float*>(host_alloc(static_cast<size_t>(total_tokens) * H_ * 4, true, &pin_seconds_));
        h_pfx_tokens_ = total_tokens;
    }
}

PrefillReport Runtime::prefill(const int32_t* tokens, const int32_t* lens, int32_t* first_ids) {
    int64_t total = 0;
    int max_len = 0;
    for (int i = 0; i < N_; ++i) {
        if (lens[i] < 1 || lens[i] >= max_ctx_)
            throw std::invalid_argument("prefill: every prompt needs 1 <= len < max_ctx");
        total += lens[i];
        max_len = std::max(max_len, lens[i]);
    }
    check_token_ids(tokens, total, V_, "prefill tokens");
    prefill_alloc(total, max_len);
    const int T = pf_T_;

    PrefillReport rep;
    rep.prompt_tokens = total;
    rep.chunk_tokens = T;
    cudaStream_t s_w = nullptr;
    ck(cudaStreamCreateWithFlags(&s_w, cudaStreamNonBlocking), "stream");
    std::vector<cudaEvent_t> owned;
    auto mk = [&](bool timing) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "event");
        owned.push_back(e);
        return e;
    };
    int32_t* h_meta = nullptr;
    int launches = 0;
    auto pl = [&](const char* what, cudaError_t e) {
        ck(e, what);
        ++launches;
    };

    cudaEvent_t e0 = mk(true), e_end = mk(true);
    ck(cudaEventRecord(e0, s_gpu_), "event");

    try {
        // ---- chunks of whole sequences, and their metadata (pinned) ----
        std::vector<Chunk> chunks;
        {
            int64_t tok = 0;
            for (int i = 0; i < N_;) {
                Chunk c;
                c.seq0 = i;
                c.tok0 = tok;
                while (i < N_ && c.tokens + lens[i] <= T) {
                    c.tokens += lens[i];
                    c.n_tiles += (lens[i] + 15) / 16;
                    tok += lens[i];
                    ++c.n_seq;
                    ++i;
                }
                chunks.push_back(c);
            }
        }
        const int nch = static_cast<int>(chunks.size());
        rep.chunks_per_layer = nch;
        const int64_t MC = pf_meta_cap_;
        ck(cudaHostAlloc(reinterpret_cast<void**>(&h_meta), static_cast<size_t>(nch) * MC * 4, 0), "meta");
        for (int ci = 0; ci < nch; ++ci) {
            const Chunk& c = chunks[ci];
            int32_t* m = h_meta + ci * MC;
            int32_t *ids = m, *tseq = m + T, *tseqg = m + 2 * T, *tpos = m + 3 * T, *srow = m + 4 * T,
                    *slen = m + 5 * T, *slast = m + 6 * T, *tiles = m + 7 * T;
            std::memcpy(ids, tokens + c.tok0, static_cast<size_t>(c.tokens) * 4);
            int r = 0, nt = 0;
            for (int j = 0; j < c.n_seq; ++j) {
                const int s = c.seq0 + j, len = lens[s];
                srow[j] = r;
                slen[j] = len;
                slast[j] = r + len - 1;
                for (int p = 0; p < len; ++p) {
                    tseq[r + p] = j;
                    tseqg[r + p] = s;
                    tpos[r + p] = p;
                }
                for (int q0 = 0; q0 < len; q0 += 16, ++nt) {
                    tiles[4 * nt] = r;
                    tiles[4 * nt + 1] = len;
                    tiles[4 * nt + 2] = q0;
                    tiles[4 * nt + 3] = 0;
                }
                r += len;
            }
        }

        // ---- weights: layer l into pool slot (l+1)&1 on s_w ----
        std::vector<cudaEvent_t> ev_w(L_), ev_layer(L_);
        for (int l = 0; l < L_; ++l) {
            ev_w[l] = mk(false);
            ev_layer[l] = mk(false);
        }
        auto upload = [&](int l) {
            const int g = l + 1, slot = slot_of(g);
            if (layer_blob_bytes_) {
                if (l >= 2) ck(cudaStreamWaitEvent(s_w, ev_layer[l - 2], 0), "wait");  // slot reuse (WAR)
                const uint8_t* src = host_blob_ + static_cast<int64_t>(l) * layer_blob_bytes_;
                if (!opt_.pin_weights) {
                    if (l >= 2) ck(cudaEventSynchronize(ev_w[l - 2]), "staging reuse");
                    uint8_t* st = staging_ + static_cast<int64_t>(slot) * layer_blob_bytes_;
                    std::memcpy(st, src, static_cast<size_t>(layer_blob_bytes_));
                    src = st;
                }
                ck(cudaMemcpyAsync(dev_pool_ + static_cast<int64_t>(slot) * layer_blob_bytes_, src,
                                   static_cast<size_t>(layer_blob_bytes_), cudaMemcpyHostToDevice, s_w),
                   "prefill weights");
                rep.h2d_weight_bytes += static_cast<double>(layer_blob_bytes_);
            }
            ck(cudaEventRecord(ev_w[l], s_w), "event");
        };
        upload(0);

        cudaEvent_t ev_loaded[2] = {mk(false), mk(false)}, ev_done[2] = {mk(false), mk(false)},
                    ev_stored[2] = {mk(false), mk(false)};
        bool used[2] = {false, false};
        // chunk ci's residual written back at layer l-1 must land before layer l reads it
        std::vector<cudaEvent_t> ev_out(nch);
        for (auto& e : ev_out) e = mk(false);
        std::vector<cudaEvent_t> busy_ev;
        const size_t kv_half = static_cast<size_t>(T) * nkv_ * d_;

        for (int l = 0; l < L_; ++l) {
            const int g = l + 1;
            const uint8_t** tab = dev_tables_ + (static_cast<size_t>(l) * 2 + slot_of(g)) * table_entries_;
            if (l + 1 < L_) upload(l + 1);
            ck(cudaStreamWaitEvent(s_gpu_, ev_w[l], 0), "wait weights");
            for (int ci = 0; ci < nch; ++ci) {
                const Chunk& c = chunks[ci];
                const int b = (l * nch + ci) & 1;
                const int Tc = c.tokens;
                float* x = pf_x_[b];
                // ---- residual in (H2D) ----
                if (used[b]) ck(cudaStreamWaitEvent(s_h2d_, ev_stored[b], 0), "wait");
                if (l > 0) {
                    ck(cudaStreamWaitEvent(s_h2d_, ev_out[ci], 0), "wait");
                    ck(cudaMemcpyAsync(x, h_pfx_ + c.tok0 * H_, static_cast<size_t>(Tc) * H_ * 4,
                                       cudaMemcpyHostToDevice, s_h2d_),
                       "prefill x in");
                    rep.h2d_bytes += static_cast<double>(Tc) * H_ * 4;
                }
                ck(cudaEventRecord(ev_loaded[b], s_h2d_), "event");
                used[b] = true;
                // ---- compute ----
                ck(cudaStreamWaitEvent(s_gpu_, ev_loaded[b], 0), "wait");
                cudaEvent_t cs = mk(true), ce = mk(true);
                busy_ev.push_back(cs);
                busy_ev.push_back(ce);
                ck(cudaEventRecord(cs, s_gpu_), "event");
                int32_t* dm = pf_meta_ + b * MC;
                ck(cudaMemcpyAsync(dm, h_meta + ci * MC, static_cast<size_t>(MC) * 4, cudaMemcpyHostToDevice, s_gpu_),
                   "prefill meta");
                rep.h2d_bytes += static_cast<double>(MC) * 4;
                const int32_t *d_ids = dm, *d_tseq = dm + T, *d_tseqg = dm + 2 * T, *d_tpos = dm + 3 * T,
                              *d_srow = dm + 4 * T, *d_slen = dm + 5 * T, *d_slast = dm + 6 * T;
                const int4* d_tiles = reinterpret_cast<const int4*>(dm + 7 * T);
                if (l == 0) pl("embed", mltk::launch_embed(d_ids, d_embed_, Tc, H_, x, s_gpu_));
                const int ncap = std::min(256, round_up(Tc, 16));
                const int nchunks = (Tc + ncap - 1) / ncap;
                // PreAttn: RMSNorm -> QKV -> rope
                pl("rmsnorm_pack", mltk::launch_rmsnorm_pack(x, d_attn_norm_[l], Tc, H_, ext_.rms_eps, pf_xn_, pf_R_, s_gpu_));
                mltk::GemmArgs a;
                a.a_table = tab + tab_qkv_;
                a.RB = W_ / 128;
                a.K = H_;
                a.b = pf_xn_;
                a.R = pf_R_;
                a.rows_dense = Tc;
                a.n_cap = ncap;
                a.n_chunks = nchunks;
                a.out_f32 = pf_y_;
                a.ldo = W_;
                codec_args(a, kWqkv);
                pl("qkv_gemm", mltk::launch_gemm(a, num_sms_, s_gpu_));
                // KV: host cache (staged, one strided DMA per sequence) or the paged
                // device pool (stored by rope_qkv itself)
                mltk::KvAppend kv;
                if (policy_.attn_on_gpu) {
                    kv.k_pool = d_kpool_;
                    kv.v_pool = d_vpool_;
                    kv.block_table = d_block_table_ + static_cast<size_t>(l) * N_ * max_pages_;
                    kv.max_pages = max_pages_;
                    kv.seq = d_tseqg;
                }
                pl("rope_qkv", mltk::launch_rope_qkv(pf_y_, 1, 0, d_tpos, d_rope_, Tc, nq_, nkv_, d_, pf_qkv_, s_gpu_,
                                                     policy_.attn_on_gpu ? &kv : nullptr));
                uint16_t* sk = pf_kst_[b];
                if (!policy_.attn_on_gpu)
                    pl("kv_stage", mltk::launch_kv_stage(pf_qkv_, W_, nq_, nkv_, d_, d_tseq, d_tpos, d_srow, d_slen,
                                                         Tc, sk, sk + kv_half, s_gpu_));
                pl("prefill_attention", mltk::launch_prefill_attention(pf_qkv_, W_, d_tiles, c.n_tiles, nq_, nkv_, d_,
                                                                       pf_xn_, pf_R_, s_gpu_));
                // PostAttn: O (+ residual) -> router -> permute -> experts -> combine
                mltk::GemmArgs o;
                o.a_table = tab + tab_o_;
                o.RB = H_ / 128;
                o.K = Ho_;
                o.b = pf_xn_;
                o.R = pf_R_;
                o.rows_dense = Tc;
                o.n_cap = ncap;
                o.n_chunks = nchunks;
                o.out_f32 = pf_h_;
                o.ldo = H_;
                o.residual = coll_ ? nullptr : x;
                o.ldr = H_;
                codec_args(o, kWo);
                pl("o_gemm", mltk::launch_gemm(o, num_sms_, s_gpu_));
                if (coll_) {
                    coll_->all_reduce_sum(pf_h_, static_cast<size_t>(Tc) * H_, s_gpu_);
                    pl("router", mltk::launch_router(pf_h_, d_ffn_norm_[l], ext_.rms_eps, nullptr, d_router_[l], Tc, H_,
                                                     E_, K_, pf_hn_, nullptr, pf_topk_, pf_topw_, s_gpu_, 1, 0, x, pf_h_));
                } else {
                    pl("router", mltk::launch_router(pf_h_, d_ffn_norm_[l], ext_.rms_eps, nullptr, d_router_[l], Tc, H_,
                                                     E_, K_, pf_hn_, nullptr, pf_topk_, pf_topw_, s_gpu_));
                }
                pl("moe_permute", mltk::launch_moe_permute(pf_topk_, pf_hn_, Tc, H_, E_, K_, d_cnt_, d_off_, pf_perm_,
                                                           pf_inv_, pf_xe_, pf_Re_, s_gpu_));
                mltk::GemmArgs gu;
                gu.a_table = tab + tab_w13_;
                gu.n_mats = 2;
                gu.G = E_;
                gu.RB = F_ / 128;
                gu.K = H_;
                gu.b = pf_xe_;
                gu.R = pf_Re_;
                gu.b_off = d_off_;
                gu.b_cnt = d_cnt_;
                gu.n_cap = ncap;
                gu.n_chunks = nchunks;  // an expert sees each token at most once
                gu.epi = mltk::kEpiSiluPacked;
                gu.out_packed = pf_inter_;
                gu.out_R = pf_Re_;
                codec_args(gu, kW1);
                pl("expert_gateup_gemm", mltk::launch_gemm(gu, num_sms_, s_gpu_));
                mltk::GemmArgs dn;
                dn.a_table = tab + tab_w2_;
                dn.G = E_;
                dn.RB = H_ / 128;
                dn.K = F_;
                dn.b = pf_inter_;
                dn.R = pf_Re_;
                dn.b_off = d_off_;
                dn.b_cnt = d_cnt_;
                dn.n_cap = ncap;
                dn.n_chunks = nchunks;
                dn.out_f32 = pf_y_;
                dn.ldo = H_;
                codec_args(dn, kW2);
                pl("expert_down_gemm", mltk::launch_gemm(dn, num_sms_, s_gpu_));
                if (coll_) {
                    pl("moe_combine", mltk::launch_moe_combine(nullptr, pf_y_, H_, pf_inv_, pf_topw_, Tc, H_, K_, x, s_gpu_));
                    coll_->all_reduce_sum(x, static_cast<size_t>(Tc) * H_, s_gpu_);
                    pl("residual_add", mltk::launch_sum_parts(x, 1, 0, pf_h_, x, static_cast<int64_t>(Tc) * H_, s_gpu_));
                } else {
                    pl("moe_combine", mltk::launch_moe_combine(pf_h_, pf_y_, H_, pf_inv_, pf_topw_, Tc, H_, K_, x, s_gpu_));
                }
                if (l == L_ - 1) {
                    // the first generated token: final norm -> lm_head -> argmax on each prompt's last row
                    for (int j0 = 0; j0 < c.n_seq; j0 += mu_) {
                        const int n = std::min(mu_, c.n_seq - j0);
                        pl("gather_rows", mltk::launch_gather_rows(x, d_slast + j0, n, H_, d_h_, s_gpu_));
                        pl("rmsnorm_pack", mltk::launch_rmsnorm_pack(d_h_, d_final_norm_, n, H_, ext_.rms_eps, d_xn_, Rmu_, s_gpu_));
                        mltk::GemmArgs lm;
                        lm.a_table = d_lm_table_;
                        lm.RB = V_ / 128;
                        lm.K = H_;
                        lm.b = d_xn_;
                        lm.R = Rmu_;
                        lm.rows_dense = n;
                        lm.n_cap = std::min(256, round_up(n, 16));
                        lm.n_chunks = (n + lm.n_cap - 1) / lm.n_cap;
                        lm.out_f32 = d_logits_;
                        lm.ldo = V_;
                        pl("lm_head_gemm", mltk::launch_gemm(lm, num_sms_, s_gpu_));
                        pl("argmax", mltk::launch_argmax(d_logits_, n, V_, d_tok_out_ + c.seq0 + j0, nullptr, s_gpu_));
                    }
                }
                ck(cudaEventRecord(ce, s_gpu_), "event");
                ck(cudaEventRecord(ev_done[b], s_gpu_), "event");
                // ---- residual + KV out (D2H) ----
                ck(cudaStreamWaitEvent(s_d2h_, ev_done[b], 0), "wait");
                if (l + 1 < L_) {
                    ck(cudaMemcpyAsync(h_pfx_ + c.tok0 * H_, x, static_cast<size_t>(Tc) * H_ * 4, cudaMemcpyDeviceToHost,
                                       s_d2h_),
                       "prefill x out");
                    rep.d2h_bytes += static_cast<double>(Tc) * H_ * 4;
                }
                if (!policy_.attn_on_gpu) {
                    const int32_t* m = h_meta + ci * MC;
                    for (int j = 0; j < c.n_seq; ++j) {
                        const int s = c.seq0 + j, len = m[5 * T + j];
                        const size_t src_off = static_cast<size_t>(m[4 * T + j]) * nkv_ * d_;
                        const size_t dst_off = ((static_cast<size_t>(l) * N_ + s) * nkv_) * max_ctx_ * d_;
                        for (int which = 0; which < 2; ++which) {
                            uint16_t* dst = (which ? h_vcache_ : h_kcache_) + dst_off;
                            ck(cudaMemcpy2DAsync(dst, static_cast<size_t>(max_ctx_) * d_ * 2, sk + which * kv_half + src_off,
                                                 static_cast<size_t>(len) * d_ * 2, static_cast<size_t>(len) * d_ * 2, nkv_,
                                                 cudaMemcpyDeviceToHost, s_d2h_),
                               "prefill kv out");
                        }
                        rep.d2h_bytes += 2.0 * len * nkv_ * d_ * 2;
                    }
                }
                ck(cudaEventRecord(ev_stored[b], s_d2h_), "event");
                ck(cudaEventRecord(ev_out[ci], s_d2h_), "event");
            }
            ck(cudaEventRecord(ev_layer[l], s_gpu_), "event");
        }
        // join the copy streams, fetch the first generated ids
        for (cudaStream_t st : {s_h2d_, s_d2h_, s_w}) {
            cudaEvent_t j = mk(false);
            ck(cudaEventRecord(j, st), "event");
            ck(cudaStreamWaitEvent(s_gpu_, j, 0), "wait");
        }
        ck(cudaMemcpyAsync(h_tok_, d_tok_out_, static_cast<size_t>(N_) * 4, cudaMemcpyDeviceToHost, s_gpu_), "ids");
        ck(cudaEventRecord(e_end, s_gpu_), "event");
        ck(cudaEventSynchronize(e_end), "prefill sync");
        std::memcpy(first_ids, h_tok_, static_cast<size_t>(N_) * 4);
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, e0, e_end), "elapsed");
        rep.seconds = ms * 1e-3;
        for (size_t i = 0; i + 1 < busy_ev.size(); i += 2) {
            float t = 0;
            ck(cudaEventElapsedTime(&t, busy_ev[i], busy_ev[i + 1]), "elapsed");
            rep.gpu_busy_seconds += t * 1e-3;
        }
    } catch (...) {
        cudaDeviceSynchronize();
        for (cudaEvent_t e : owned) cudaEventDestroy(e);
        if (h_meta) cudaFreeHost(h_meta);
        cudaStreamDestroy(s_w);
        throw;
    }
    for (cudaEvent_t e : owned) cudaEventDestroy(e);
    cudaFreeHost(h_meta);
    cudaStreamDestroy(s_w);
    rep.h2d_bytes += rep.h2d_weight_bytes;  // token ids ride in the chunk metadata
    rep.d2h_bytes += static_cast<double>(N_) * 4;
    rep.gpu_launches = launches;
    rep.tokens_per_second = static_cast<double>(total) / rep.seconds;
    for (int i = 0; i < N_; ++i) pos_[i] = lens[i];
    return rep;
}

}  // namespace mlt
