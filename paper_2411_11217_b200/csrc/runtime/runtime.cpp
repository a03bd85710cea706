// Runtime construction (arena, weight catalog + residency, paged weight
// store, activation buffers) and the per-task actions the CGOPipe executor
// runs.  See runtime.hpp and DESIGN.md §3-§5.
#include "runtime.hpp"

#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../capi/status.hpp"
#include "../kernels/common.cuh"
#include "../kernels/kernels.hpp"
#include "host_layout.hpp"
#include "weight_codec.hpp"
#include "runtime_util.hpp"

namespace mlt {

namespace {
using detail::ck;
using detail::now_s;
using detail::round_up;
}  // namespace

namespace detail {
// Large host buffers: 2 MiB-aligned, transparent huge pages, first-touched
// in parallel, then page-locked with cudaHostRegister (measured on the GPU
// box: ~0.1 s/GB vs ~0.4 s/GB for cudaHostAlloc; tools/pin_probe.cu).
uint8_t* host_alloc(size_t bytes, bool pin, double* pin_seconds) {
    const size_t align = 2u << 20;
    bytes = (bytes + align - 1) / align * align;
    void* p = std::aligned_alloc(align, bytes);
    if (!p) throw std::bad_alloc();
    madvise(p, bytes, MADV_HUGEPAGE);
    uint8_t* b = static_cast<uint8_t*>(p);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < static_cast<int64_t>(bytes); i += 4096) b[i] = 0;
    if (pin) {
        const double t = now_s();
        ck(cudaHostRegister(p, bytes, cudaHostRegisterDefault), "cudaHostRegister");
        if (pin_seconds) *pin_seconds += now_s() - t;
    }
    return b;
}

void host_free(void* p, bool pinned) {
    if (!p) return;
    if (pinned) cudaHostUnregister(p);
    std::free(p);
}
}  // namespace detail
using detail::host_alloc;
using detail::host_free;

// ---------------------------------------------------------------------------
Arena::Arena(size_t bytes) : cap_(bytes) {
    ck(cudaMalloc(&base_, bytes), "arena cudaMalloc (budget)");
}
Arena::~Arena() {
    if (base_) cudaFree(base_);
}
void* Arena::alloc(size_t bytes, const char* what) {
    const size_t off = (used_ + 1023) & ~static_cast<size_t>(1023);
    if (off + bytes > cap_)
        throw BudgetError(std::string("device budget exceeded allocating ") + what + " (" +
                          std::to_string(bytes) + " B; used " + std::to_string(off) + " of " +
                          std::to_string(cap_) + ")");
    used_ = off + bytes;
    log_ += std::string(what) + "=" + std::to_string(bytes) + ";";
    return base_ + off;
}

// ---------------------------------------------------------------------------
Runtime::Runtime(const lightplan::ModelSpec& model, const ModelExt& ext,
                 const lightplan::Policy& policy, const RuntimeOptions& opt)
    : model_(model), ext_(ext), policy_(policy), opt_(opt) {
    auto issues = lightplan::validate(model);
    auto pi = lightplan::validate(policy);
    issues.insert(issues.end(), pi.begin(), pi.end());
    if (!issues.empty()) throw std::invalid_argument(lightplan::format_issues(issues));
    N_ = static_cast<int>(policy.batch);
    mu_ = static_cast<int>(policy.micro_batch);
    M_ = static_cast<int>(policy.micro_batch_count());
    H_ = static_cast<int>(model.hidden_dim);
    F_ = static_cast<int>(model.ffn_dim);
    E_ = static_cast<int>(model.experts);
    K_ = static_cast<int>(model.top_k);
    nq_ = static_cast<int>(model.q_heads);
    nkv_ = static_cast<int>(model.kv_heads);
    d_ = static_cast<int>(model.head_dim());
    W_ = (nq_ + 2 * nkv_) * d_;
    V_ = ext.vocab;
    L_ = static_cast<int>(model.layers);
    shard_ = make_shard(model, opt.tp_rank, opt.tp_size);
    // this rank's slice of every sharded matrix (exec_plan.cpp shard_map): QKV, O, W1/W3, W2
    maps_[0] = shard_map(model, shard_, kWqkv);
    maps_[1] = shard_map(model, shard_, kWo);
    maps_[2] = shard_map(model, shard_, kW1);
    maps_[3] = shard_map(model, shard_, kW2);
    nq_ = static_cast<int>(shard_.q_heads);
    nkv_ = static_cast<int>(shard_.kv_heads);
    F_ = static_cast<int>(shard_.ffn);
    W_ = static_cast<int>(shard_.qkv_rows);
    Ho_ = static_cast<int>(shard_.o_k);
    if (model.weight_dtype_bytes != 2 || model.kv_dtype_bytes != 2)
        throw std::invalid_argument("runtime supports bf16 weights and KV (dt_w = dt_kv = 2)");
    if (H_ % 256 || F_ % 128 || W_ % 128 || V_ % 128 || d_ != 128 || E_ > 64 || K_ > 8)
        throw std::invalid_argument("shape: need h1 % 256, h2 % 128, vocab % 128, head_dim 128, n_e <= 64, k <= 8");
    if (!policy.ffn_on_gpu) throw lightplan::sim::UnsupportedCombinationError("F_g = 0 is not a B200 path");
    if (policy.attn_on_gpu && policy.kv_on_gpu < 1.0)
        throw lightplan::sim::UnsupportedCombinationError("A_g = 1 requires r_c = 1 (resident paged KV) in this build");
    if (opt.schedule < -1 || opt.schedule > 3) throw std::invalid_argument("schedule must be -1 or 0..3");
    schedule_kind();  // rejects S4 without A_g / CGOPipe,S2,S3 with A_g (pipesim.cpp:283-290)
    if (opt.max_ctx <= 0) throw std::invalid_argument("max_ctx must be > 0");
    {   // GQA group size this rank's attention kernels support (host: register
        // blocking up to 16 heads per kv head; GPU decode: G in {1,2,4,6,8};
        // the GPU prefill: G <= 8)
        const int G = nkv_ > 0 ? nq_ / nkv_ : 0;
        if (G < 1 || nq_ % nkv_) throw std::invalid_argument("q_heads / kv_heads must be a positive integer");
        if (!policy.attn_on_gpu && G > 16)
            throw std::invalid_argument("host attention supports q_heads / kv_heads <= 16 (got " + std::to_string(G) + ")");
        if (policy.attn_on_gpu && G != 1 && G != 2 && G != 4 && G != 6 && G != 8)
            throw std::invalid_argument("GPU decode attention supports q_heads / kv_heads in {1, 2, 4, 6, 8} (got " +
                                        std::to_string(G) + ")");
    }
    max_ctx_ = opt.max_ctx;
    Rmu_ = round_up(mu_, 16);
    // encoded weights: the tcgen05 GEMM with the A operand decoded into tensor
    // memory (codec 3, row-plane tiles, three decoupled rings): expert FFN at
    // mu = 64 391 us vs 451 us for the in-smem decoder (codec 1) and 450 us for
    // raw bf16 (profiles/r02s2_codec_engines.txt).  MLT_CODEC_MODE=1 selects the
    // in-smem decoder, MLT_CODEC_MODE=2 the register-decode mma.sync GEMM
    // (fragment-order tiles, while a micro-batch fits its 64-token chunks).
    // Codec 4 (the default) is the same engine on the 3-bit code: ~11600 B per
    // tile instead of 12432 (weight_codec.hpp); MLT_CODEC_MODE=3 keeps the
    // 4-bit code.  Weights the 3-bit code holds badly (see below) fall back to
    // codec 3 after the scan (scan_raw_blocks).
    codec_mode_ = 0;
    if (opt.weight_codec) {
        const char* m = std::getenv("MLT_CODEC_MODE");
        codec_mode_ = (m && m[0] == '2' && Rmu_ <= 64) ? 2 : (m && m[0] == '1') ? 1 : (m && m[0] == '3') ? 3 : 4;
    }
    Re_ = round_up(mu_ * K_ + 16 * E_, 16);
    ncap_ = std::min(256, Rmu_);
    ncap_e_ = std::min(128, Rmu_);  // per-expert tiles: 4+ smem stages; m_e > 128 loops in-tile
    pos_.assign(N_, 0);

    ck(cudaSetDevice(opt.device), "cudaSetDevice");
    ck(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, opt.device), "sm count");
    ck(cudaStreamCreateWithFlags(&s_gpu_, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&s_h2d_, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&s_d2h_, cudaStreamNonBlocking), "stream");
    if (opt.tp_size > 1) {
        if (opt.tp_shard_only)
            coll_ = make_elided_collective(opt.tp_rank, opt.tp_size);
        else if (opt.collective == 1)  // host-staged: the rendezvous name travels in nccl_id
            coll_ = make_host_collective(std::string(reinterpret_cast<const char*>(opt.nccl_id),
                                                     strnlen(reinterpret_cast<const char*>(opt.nccl_id), 127)),
                                         opt.tp_rank, opt.tp_size, static_cast<size_t>(mu_) * H_);
        else if (opt.collective == 0)
            coll_ = make_nccl_collective(opt.nccl_id, opt.tp_rank, opt.tp_size, opt.device);
        else
            throw std::invalid_argument("collective must be 0 (NCCL) or 1 (host-staged)");
    }
    arena_ = std::make_unique<Arena>(static_cast<size_t>(opt.budget_bytes));
    // every block of every layer is test-encoded once when some tile may not
    // fit: caller weights (any code), and the 3-bit code even for the
    // synthetic weights (~14 of its 48 escapes per tile on average)
    if (opt.weight_codec && (opt.weight_fn || codec_mode_ == 4)) {
        const char* f = std::getenv("MLT_CODEC_FORCE_RAW");
        if (!(f && f[0] == '1')) {
            scan_raw_blocks();
            int raw = 0, cap = 0;
            for (uint8_t b : raw_mask_) raw += b;
            for (int k = 0; k < 16; ++k) cap = std::max(cap, c4_cap_[k]);
            // the 3-bit code pays while its tile stays clearly smaller than the
            // 4-bit code's 12432 B and hard escapes stay rare: fall back when
            // more than 5 % of the blocks would be raw or a kind needs more
            // than 128 entries per tile (11936 B; heavy-tailed weights: ~110
            // entries, ~30 of them hard escapes)
            if (codec_mode_ == 4 && (raw * 20 > static_cast<int>(raw_mask_.size()) || cap > 128)) {
                codec_mode_ = 3;
                scan_raw_blocks();
            }
        }
    }
    build_catalog();
    allocate();
    generate_weights();
    prefill_task_events(32);  // a 32-step decode's task events, outside every decode call
}

Runtime::~Runtime() {
    cudaDeviceSynchronize();
    for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
    for (cudaEvent_t e : task_ev_) cudaEventDestroy(e);
    host_free(host_blob_, host_blob_pinned_);
    host_free(staging_, true);
    if (h_qkv_) cudaFreeHost(h_qkv_);
    if (h_attn_) cudaFreeHost(h_attn_);
    if (h_tok_) cudaFreeHost(h_tok_);
    if (h_cap_hn_) cudaFreeHost(h_cap_hn_);
    if (h_cap_topk_) cudaFreeHost(h_cap_topk_);
    if (h_cap_topw_) cudaFreeHost(h_cap_topw_);
    host_free(h_kcache_, true);
    host_free(h_vcache_, true);
    host_free(h_pfx_, true);
    arena_.reset();
    if (s_gpu_) cudaStreamDestroy(s_gpu_);
    if (s_h2d_) cudaStreamDestroy(s_h2d_);
    if (s_d2h_) cudaStreamDestroy(s_d2h_);
}

cudaStream_t Runtime::stream(lightplan::sim::Resource r) const {
    switch (r) {
        case lightplan::sim::Resource::Gpu: return s_gpu_;
        case lightplan::sim::Resource::HostToDevice: return s_h2d_;
        case lightplan::sim::Resource::DeviceToHost: return s_d2h_;
        default: return nullptr;
    }
}

// Residency split and blob layout: exec_plan.cpp build_catalog.
void Runtime::build_catalog() {
    // codec: per-block raw fallback mask (test knob MLT_CODEC_FORCE_RAW=1 stores
    // every block raw, which must decode bit-identically to the encoded run)
    if (opt_.weight_codec) {
        const char* f = std::getenv("MLT_CODEC_FORCE_RAW");
        if (f && f[0] == '1')
            raw_mask_.assign(mlt::build_catalog(model_, policy_, shard_, true).blocks.size(), 1);
    }
    int kind_tile[16];
    for (int k = 0; k < 16; ++k) kind_tile[k] = codec_mode_ == 4 ? c4_tile_[k] : codec_tile_bytes(codec_mode_);
    cat_ = mlt::build_catalog(model_, policy_, shard_, opt_.weight_codec, raw_mask_.empty() ? nullptr : &raw_mask_,
                              kind_tile);
    any_raw_ = false;
    for (const auto& b : cat_.blocks) any_raw_ = any_raw_ || b.raw;
    layer_res_bytes_ = cat_.resident_bytes;
    layer_blob_bytes_ = cat_.blob_bytes;
    achieved_rw_ = cat_.achieved_rw;
}

void Runtime::allocate() {
    Arena& A = *arena_;
    const int64_t T = static_cast<int64_t>(N_);
    // weights
    if (layer_res_bytes_) dev_res_ = static_cast<uint8_t*>(A.alloc(L_ * layer_res_bytes_, "resident_weights"));
    if (layer_blob_bytes_) dev_pool_ = static_cast<uint8_t*>(A.alloc(2 * layer_blob_bytes_, "page_pool"));
    d_embed_ = static_cast<uint16_t*>(A.alloc(static_cast<size_t>(V_) * H_ * 2, "embed"));
    d_lm_ = static_cast<uint16_t*>(A.alloc(static_cast<size_t>(V_) * H_ * 2, "lm_head"));
    d_final_norm_ = static_cast<uint16_t*>(A.alloc(H_ * 2, "final_norm"));
    for (int l = 0; l < L_; ++l) {
        d_attn_norm_.push_back(static_cast<uint16_t*>(A.alloc(H_ * 2, "attn_norm")));
        d_ffn_norm_.push_back(static_cast<uint16_t*>(A.alloc(H_ * 2, "ffn_norm")));
        d_router_.push_back(static_cast<uint16_t*>(A.alloc(static_cast<size_t>(E_) * H_ * 2, "router")));
    }
    tab_qkv_ = 0;
    tab_o_ = tab_qkv_ + W_ / 128;
    tab_w13_ = tab_o_ + H_ / 128;
    tab_w2_ = tab_w13_ + 2 * E_ * (F_ / 128);
    table_entries_ = tab_w2_ + E_ * (H_ / 128);
    dev_tables_ = static_cast<const uint8_t**>(A.alloc(sizeof(void*) * L_ * 2 * table_entries_, "page_tables"));
    d_lm_table_ = static_cast<const uint8_t**>(A.alloc(sizeof(void*) * (V_ / 128), "lm_table"));
    d_rope_ = static_cast<float2*>(A.alloc(sizeof(float2) * max_ctx_ * (d_ / 2), "rope"));
    // activations
    d_x_ = static_cast<float*>(A.alloc(T * H_ * 4, "x"));
    d_qkv_bf16_ = static_cast<uint16_t*>(A.alloc(static_cast<size_t>(M_) * mu_ * W_ * 2, "qkv_bf16"));
    d_attn_in_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(M_) * Rmu_ * Ho_ * 2, "attn_in"));
    if (coll_) d_cbuf_ = static_cast<float*>(A.alloc(static_cast<size_t>(mu_) * H_ * 4, "tp_combine"));
    // one normed-activation operand per micro-batch: the fused combine+norm of
    // PostAttn(layer l, mb) produces PreAttn(layer l+1, mb)'s operand, and
    // other micro-batches' PreAttn run in between (CGOPipe order)
    d_xn_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(M_) * Rmu_ * H_ * 2, "xn"));
    d_qkv_f32_ = static_cast<float*>(A.alloc(static_cast<size_t>(kMaxSplits) * Rmu_ * W_ * 4, "qkv_f32"));
    d_h_ = static_cast<float*>(A.alloc(static_cast<size_t>(mu_) * H_ * 4, "h"));
    d_hparts_ = static_cast<float*>(A.alloc(static_cast<size_t>(kMaxSplits) * mu_ * H_ * 4, "h_parts"));
    d_hn_ = static_cast<uint16_t*>(A.alloc(static_cast<size_t>(mu_) * H_ * 2, "hn"));
    d_topk_ = static_cast<int32_t*>(A.alloc(mu_ * K_ * 4, "topk"));
    d_topw_ = static_cast<float*>(A.alloc(mu_ * K_ * 4, "topw"));
    d_cnt_ = static_cast<int32_t*>(A.alloc(E_ * 4, "counts"));
    d_off_ = static_cast<int32_t*>(A.alloc((E_ + 1) * 4, "offsets"));
    d_perm_ = static_cast<int32_t*>(A.alloc(Re_ * 4, "perm"));
    d_inv_ = static_cast<int32_t*>(A.alloc(mu_ * K_ * 4, "inv"));
    d_xe_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(Re_) * H_ * 2, "expert_in"));
    d_inter_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(Re_) * F_ * 2, "expert_inter"));
    // expert down GEMM split-K: with encoded weights each SM's tile rate is
    // bound by its decoders, so the SMs idle in a partial last wave are lost
    // time (8x7B: 8 x 32 row blocks = 1.73 waves of 148 SMs -> 86 % fill;
    // 4 splits: 6.92 waves -> 99 %); bf16 tiles are HBM-bound and need none
    down_splits_ = opt_.expert_down_splits;
    if (down_splits_ <= 0) {
        down_splits_ = 1;
        if (opt_.weight_codec) {
            const int tiles = E_ * (H_ / 128);
            double best = 0;
            for (int s = 1; s <= 8 && (F_ / 64) / s >= 8; ++s) {
                const double waves = static_cast<double>(tiles) * s / gemm_slots();
                const double fill = waves / std::ceil(waves);
                if (fill > best + 1e-9) best = fill, down_splits_ = s;
            }
        }
    }
    if (down_splits_ > 8 || (F_ / 64) < down_splits_) throw std::invalid_argument("expert_down_splits must be <= 8 and <= h2/64");
    d_y_ = static_cast<float*>(A.alloc(static_cast<size_t>(down_splits_) * Re_ * H_ * 4, "expert_out"));
    // gate/up stream-K tail (gemm_tc.cu): parts of the partial last wave's tiles
    d_sk_scratch_ = static_cast<float*>(A.alloc(static_cast<size_t>(num_sms_) * 2 * Rmu_ * 128 * 4, "sk_scratch"));
    d_sk_count_ = static_cast<unsigned long long*>(A.alloc(static_cast<size_t>(num_sms_) * 8, "sk_count"));
    ck(cudaMemset(d_sk_count_, 0, static_cast<size_t>(num_sms_) * 8), "sk_count");
    d_logits_ = static_cast<float*>(A.alloc(static_cast<size_t>(mu_) * V_ * 4, "logits"));
    d_tok_in_ = static_cast<int32_t*>(A.alloc(static_cast<size_t>(max_steps_) * N_ * 4, "tok_in"));
    d_tok_out_ = static_cast<int32_t*>(A.alloc(static_cast<size_t>(max_steps_) * N_ * 4, "tok_out"));
    d_pos_ = static_cast<int32_t*>(A.alloc(static_cast<size_t>(max_steps_) * N_ * 4 * 2, "pos_ctx"));
    d_seq_ = static_cast<int32_t*>(A.alloc(static_cast<size_t>(N_) * 4, "seq"));
    ktime_cap_ = max_steps_ * L_ * M_ * 4 + 16;
    d_ktime_ = static_cast<unsigned long long*>(A.alloc(static_cast<size_t>(ktime_cap_) * 16, "kernel_timers"));
    if (policy_.attn_on_gpu) {
        max_pages_ = (max_ctx_ + page_ - 1) / page_;
        const size_t pages = static_cast<size_t>(L_) * N_ * max_pages_;
        const size_t bytes = pages * nkv_ * page_ * d_ * 2;
        d_kpool_ = static_cast<uint16_t*>(A.alloc(bytes, "kv_pool_k"));
        d_vpool_ = static_cast<uint16_t*>(A.alloc(bytes, "kv_pool_v"));
        d_block_table_ = static_cast<int32_t*>(A.alloc(pages * 4, "block_table"));
        d_attn_gpu_ = static_cast<uint8_t*>(A.alloc(static_cast<size_t>(Rmu_) * Ho_ * 2, "attn_gpu"));

        std::vector<int32_t> bt(pages);
        for (size_t i = 0; i < pages; ++i) bt[i] = static_cast<int32_t>(i);  // per (layer, seq) page runs
        ck(cudaMemcpy(d_block_table_, bt.data(), pages * 4, cudaMemcpyHostToDevice), "block table");
    }
    std::vector<int32_t> seq(N_);
    for (int i = 0; i < N_; ++i) seq[i] = i;
    ck(cudaMemcpy(d_seq_, seq.data(), N_ * 4, cudaMemcpyHostToDevice), "seq");
    std::vector<float> rope(static_cast<size_t>(max_ctx_) * d_);
    for (int p = 0; p < max_ctx_; ++p)
        for (int i = 0; i < d_ / 2; ++i) {
            const double inv = std::pow(static_cast<double>(ext_.rope_theta), -2.0 * i / static_cast<double>(d_));
            const double ang = static_cast<double>(p) * inv;
            rope[(static_cast<size_t>(p) * (d_ / 2) + i) * 2] = static_cast<float>(std::cos(ang));
            rope[(static_cast<size_t>(p) * (d_ / 2) + i) * 2 + 1] = static_cast<float>(std::sin(ang));
        }
    ck(cudaMemcpy(d_rope_, rope.data(), rope.size() * 4, cudaMemcpyHostToDevice), "rope");

    // host side
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_qkv_), static_cast<size_t>(M_) * mu_ * W_ * 2, 0), "h_qkv");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_attn_), static_cast<size_t>(M_) * Rmu_ * Ho_ * 2, 0), "h_attn");
    std::memset(h_attn_, 0, static_cast<size_t>(M_) * Rmu_ * Ho_ * 2);
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_tok_), static_cast<size_t>(max_steps_) * N_ * 4 * 4, 0), "h_tok");
    if (!policy_.attn_on_gpu) {
        const size_t kv = static_cast<size_t>(L_) * N_ * nkv_ * max_ctx_ * d_;
        // page-locked: the GPU prefill writes the prompt KV here by DMA
        h_kcache_ = reinterpret_cast<uint16_t*>(host_alloc(kv * 2, true, &pin_seconds_));
        h_vcache_ = reinterpret_cast<uint16_t*>(host_alloc(kv * 2, true, &pin_seconds_));
    }
}

const uint16_t* Runtime::ext_tensor(int l, int kind, int expert) const {
    const uint16_t* p = opt_.weight_fn(opt_.weight_ctx, l, kind, expert);
    if (!p)
        throw std::invalid_argument("weights: no tensor for layer " + std::to_string(l) + " kind " +
                                    std::to_string(kind) + " expert " + std::to_string(expert));
    return p;
}

void Runtime::packed_block(int l, const WeightBlock& b, uint16_t* dst) const {
    const ShardMap& sm = maps_[b.kind == kWqkv ? 0 : b.kind == kWo ? 1 : b.kind == kW2 ? 3 : 2];
    if (opt_.weight_fn)
        pack_shard_rows(ext_tensor(l, b.kind, b.expert), sm.k_global, sm.rows.data(), sm.col0, b.K, b.rb * 128,
                        (b.rb + 1) * 128, dst);
    else
        synth_shard_packed(ext_.seed, tensor_id(l, b.kind, b.expert), sm.k_global, sm.rows.data(), sm.col0, b.K,
                           b.rb * 128, (b.rb + 1) * 128, sm.scale, dst);
}

void Runtime::plain_tensor(int l, int kind, int64_t n, float scale, bool is_norm, uint16_t* dst) const {
    if (opt_.weight_fn)
        std::memcpy(dst, ext_tensor(l, kind, 0), static_cast<size_t>(n) * 2);
    else
        synth_bf16(ext_.seed, tensor_id(l, kind, 0), 0, n, scale, is_norm, dst);
}

// Caller weights with the codec: a 128-row block whose tiles the code cannot
// hold (more than 31 escapes in a tile: heavy tails, outlier rows) is stored
// raw in every layer (one catalog layout for all layers, so the page pool
// and page table stay uniform).  Synthetic weights always fit.
void Runtime::scan_raw_blocks() {
    const Catalog probe = mlt::build_catalog(model_, policy_, shard_, true);
    raw_mask_.assign(probe.blocks.size(), 0);
    const bool c4 = codec_mode_ == 4;
    // codec 4: the largest records + escapes count of any tile per block, over all layers
    std::vector<int> need(probe.blocks.size(), 0);
    std::vector<uint16_t> tmp;
    for (int l = 0; l < L_; ++l)
        for (size_t i = 0; i < probe.blocks.size(); ++i) {
            if (raw_mask_[i]) continue;
            const WeightBlock& b = probe.blocks[i];
            tmp.resize(static_cast<size_t>(128) * b.K);
            packed_block(l, b, tmp.data());
            const int tiles = static_cast<int>(b.K / 64);
            int bad = 0, most = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad) reduction(max : most)
            for (int t = 0; t < tiles; ++t) {
                uint8_t out[codec4_tile_bytes(kCodec4CapLimit) > kCodecTileBytes ? codec4_tile_bytes(kCodec4CapLimit)
                                                                                 : kCodecTileBytes];
                const uint8_t* src = reinterpret_cast<const uint8_t*>(tmp.data()) +
                                     static_cast<size_t>(t) * mltk::kATileBytes;
                int n = 0;
                bad += (c4 ? codec4_encode_rows_tile(src, out, kCodec4CapLimit, &n) : codec_encode_tile(src, out)) ? 0 : 1;
                most = std::max(most, n);
            }
            if (bad) raw_mask_[i] = 1;
            need[i] = std::max(need[i], most);
        }
    if (!c4) return;
    // per weight kind (W1 and W3 share the gate/up GEMM): the capacity of its
    // fullest coded tile, rounded up to a multiple of 4 (16-byte tiles)
    for (int k = 0; k < 16; ++k) c4_cap_[k] = 0;
    for (size_t i = 0; i < probe.blocks.size(); ++i)
        if (!raw_mask_[i]) {
            const int k = probe.blocks[i].kind == kW3 ? kW1 : probe.blocks[i].kind;
            c4_cap_[k] = std::max(c4_cap_[k], need[i]);
        }
    c4_cap_[kW3] = c4_cap_[kW1];
    for (int k = 0; k < 16; ++k) {
        c4_cap_[k] = (c4_cap_[k] + 3) & ~3;
        c4_tile_[k] = codec4_tile_bytes(c4_cap_[k]);
    }
}

void Runtime::generate_weights() {
    const double t0 = now_s();
    const uint64_t seed = ext_.seed;
    const double sH = 1.0 / std::sqrt(static_cast<double>(H_));
    host_blob_pinned_ = opt_.pin_weights != 0;
    if (layer_blob_bytes_) {
        host_blob_ = host_alloc(static_cast<size_t>(L_) * layer_blob_bytes_, host_blob_pinned_, &pin_seconds_);
        if (!opt_.pin_weights) staging_ = host_alloc(2 * static_cast<size_t>(layer_blob_bytes_), true, &pin_seconds_);
    }
    std::vector<uint8_t> res(static_cast<size_t>(layer_res_bytes_));
    std::vector<uint16_t> tmp_block;
    std::vector<const uint8_t*> tab(static_cast<size_t>(L_) * 2 * table_entries_);
    for (int l = 0; l < L_; ++l) {
        int idx_qkv = 0, idx_o = 0;
        for (const auto& b : cat_.blocks) {
            uint8_t* dst = b.resident ? res.data() + b.offset
                                      : host_blob_ + static_cast<int64_t>(l) * layer_blob_bytes_ + b.offset;
            if (!opt_.weight_codec || (b.raw && codec_mode_ != 2)) {  // packed bf16 tiles
                packed_block(l, b, reinterpret_cast<uint16_t*>(dst));
            } else if (b.raw) {  // codec 2 raw fallback: fragment-order bf16 tiles
                tmp_block.resize(static_cast<size_t>(128) * b.K);
                packed_block(l, b, tmp_block.data());
                const int tiles = static_cast<int>(b.K / 64);
#pragma omp parallel for schedule(static)
                for (int t = 0; t < tiles; ++t)
                    frag_from_packed(reinterpret_cast<const uint8_t*>(tmp_block.data()) +
                                         static_cast<size_t>(t) * mltk::kATileBytes,
                                     reinterpret_cast<uint16_t*>(dst + static_cast<size_t>(t) * mltk::kATileBytes));
            } else {  // packed bf16 tiles -> encoded tiles (lossless, weight_codec.hpp)
                tmp_block.resize(static_cast<size_t>(128) * b.K);
                packed_block(l, b, tmp_block.data());
                const int tiles = static_cast<int>(b.K / 64);
                int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
                for (int t = 0; t < tiles; ++t)
                    {
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(tmp_block.data()) +
                                         static_cast<size_t>(t) * mltk::kATileBytes;
                    uint8_t* out = dst + static_cast<size_t>(t) * (codec_mode_ == 4 ? c4_tile_[b.kind]
                                                                                 : codec_tile_bytes(codec_mode_));
                    bad += (codec_mode_ == 2   ? codec_encode_frag_tile(src, out)
                            : codec_mode_ == 3 ? codec_encode_rows_tile(src, out)
                            : codec_mode_ == 4 ? codec4_encode_rows_tile(src, out, c4_cap_[b.kind])
                                               : codec_encode_tile(src, out))
                               ? 0
                               : 1;
                }
                if (bad)  // scanned (scan_raw_blocks) unless the code always fits (synthetic, 4-bit)
                    throw std::invalid_argument("weight_codec: a weight tile does not fit the code");
            }
            int entry;
            switch (b.kind) {
                case kWqkv: entry = tab_qkv_ + idx_qkv++; break;
                case kWo: entry = tab_o_ + idx_o++; break;
                case kW1: entry = tab_w13_ + b.expert * (F_ / 128) + b.rb; break;
                case kW3: entry = tab_w13_ + E_ * (F_ / 128) + b.expert * (F_ / 128) + b.rb; break;
                default: entry = tab_w2_ + b.expert * (H_ / 128) + b.rb; break;
            }
            for (int slot = 0; slot < 2; ++slot) {
                const uint8_t* p = b.resident ? dev_res_ + static_cast<int64_t>(l) * layer_res_bytes_ + b.offset
                                              : dev_pool_ + static_cast<int64_t>(slot) * layer_blob_bytes_ + b.offset;
                if (b.raw) p += 1;  // tag: raw fallback block of an encoded model (gemm_tc / gemm_codec untag)
                tab[(static_cast<size_t>(l) * 2 + slot) * table_entries_ + entry] = p;
            }
        }
        if (layer_res_bytes_)
            ck(cudaMemcpy(dev_res_ + static_cast<int64_t>(l) * layer_res_bytes_, res.data(), layer_res_bytes_,
                          cudaMemcpyHostToDevice),
               "resident upload");
        std::vector<uint16_t> v(static_cast<size_t>(E_) * H_);
        plain_tensor(l, kRouter, static_cast<int64_t>(E_) * H_, static_cast<float>(sH), false, v.data());
        ck(cudaMemcpy(d_router_[l], v.data(), v.size() * 2, cudaMemcpyHostToDevice), "router");
        plain_tensor(l, kAttnNorm, H_, 0.f, true, v.data());
        ck(cudaMemcpy(d_attn_norm_[l], v.data(), H_ * 2, cudaMemcpyHostToDevice), "attn_norm");
        plain_tensor(l, kFfnNorm, H_, 0.f, true, v.data());
        ck(cudaMemcpy(d_ffn_norm_[l], v.data(), H_ * 2, cudaMemcpyHostToDevice), "ffn_norm");
    }
    ck(cudaMemcpy(dev_tables_, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice), "tables");
    {
        std::vector<uint16_t> big(static_cast<size_t>(V_) * H_);
        plain_tensor(-1, kEmbed, static_cast<int64_t>(V_) * H_, 1.0f, false, big.data());
        ck(cudaMemcpy(d_embed_, big.data(), big.size() * 2, cudaMemcpyHostToDevice), "embed");
        const float s_lm = static_cast<float>(static_cast<double>(ext_.lm_head_scale) * sH);
        if (opt_.weight_fn)
            pack_weight(ext_tensor(-1, kLmHead, 0), V_, H_, big.data());
        else
            synth_bf16_packed(seed, tensor_id(-1, kLmHead, 0), V_, H_, 0, V_, s_lm, big.data());
        ck(cudaMemcpy(d_lm_, big.data(), big.size() * 2, cudaMemcpyHostToDevice), "lm_head");
        std::vector<const uint8_t*> lt(V_ / 128);
        for (int rb = 0; rb < V_ / 128; ++rb)
            lt[rb] = reinterpret_cast<const uint8_t*>(d_lm_) + static_cast<int64_t>(rb) * 128 * H_ * 2;
        ck(cudaMemcpy(d_lm_table_, lt.data(), lt.size() * sizeof(void*), cudaMemcpyHostToDevice), "lm table");
        std::vector<uint16_t> g(H_);
        plain_tensor(-1, kFinalNorm, H_, 0.f, true, g.data());
        ck(cudaMemcpy(d_final_norm_, g.data(), H_ * 2, cudaMemcpyHostToDevice), "final_norm");
    }
    gen_seconds_ = now_s() - t0;
}

void Runtime::prefill_synthetic(int prompt_len, uint64_t seed) {
    if (prompt_len < 0 || prompt_len >= max_ctx_) throw std::invalid_argument("prompt_len out of range");
    const int nkd = nkv_ * d_;
    std::vector<uint16_t> tmp;
    for (int l = 0; l < L_; ++l)
        for (int which = 0; which < 2; ++which) {
            const uint64_t key = mix64(seed ^ mix64(tensor_id(l, kKCache + which, 0)));
            if (!policy_.attn_on_gpu) {
                uint16_t* dst = which ? h_vcache_ : h_kcache_;
#pragma omp parallel for collapse(2) schedule(static)
                for (int s = 0; s < N_; ++s)
                    for (int h = 0; h < nkv_; ++h)
                        for (int p = 0; p < prompt_len; ++p)
                            for (int i = 0; i < d_; ++i) {
                                const uint64_t idx = ((static_cast<uint64_t>(s) << 20) | static_cast<uint64_t>(p)) * nkd + h * d_ + i;
                                const uint64_t hv = mix64(key + idx);
                                const float r = 2.0f * (static_cast<float>(hv >> 40) * 0x1p-24f) - 1.0f;
                                dst[(((static_cast<size_t>(l) * N_ + s) * nkv_ + h) * max_ctx_ + p) * d_ + i] = f32_to_bf16(r);
                            }
            } else {
                // paged device cache: page id = (l*N + s)*max_pages + p/page, [nkv][page][d]
                // with the token-row swizzle of common.cuh kv_page_off
                const size_t per_seq = static_cast<size_t>(max_pages_) * nkv_ * page_ * d_;
                tmp.assign(per_seq * N_, 0);
#pragma omp parallel for collapse(2) schedule(static)
                for (int s = 0; s < N_; ++s)
                    for (int h = 0; h < nkv_; ++h)
                        for (int p = 0; p < prompt_len; ++p)
                            for (int i = 0; i < d_; ++i) {
                                const uint64_t idx = ((static_cast<uint64_t>(s) << 20) | static_cast<uint64_t>(p)) * nkd + h * d_ + i;
                                const uint64_t hv = mix64(key + idx);
                                const float r = 2.0f * (static_cast<float>(hv >> 40) * 0x1p-24f) - 1.0f;
                                const size_t page = p / page_;
                                tmp[static_cast<size_t>(s) * per_seq + (page * nkv_ + h) * page_ * d_ +
                                    mltk::kv_page_off(p % page_, i)] = f32_to_bf16(r);
                            }
                uint16_t* pool = which ? d_vpool_ : d_kpool_;
                ck(cudaMemcpy(pool + static_cast<size_t>(l) * N_ * per_seq, tmp.data(), tmp.size() * 2,
                              cudaMemcpyHostToDevice),
                   "kv prefill");
            }
        }
    std::fill(pos_.begin(), pos_.end(), prompt_len);
}

void Runtime::set_positions(const int32_t* pos) {
    for (int i = 0; i < N_; ++i) {
        if (pos[i] < 0 || pos[i] >= max_ctx_) throw std::invalid_argument("position out of range");
        pos_[i] = pos[i];
    }
}

void Runtime::read_residual(float* out) {
    ck(cudaStreamSynchronize(s_gpu_), "sync");
    ck(cudaMemcpy(out, d_x_, static_cast<size_t>(N_) * H_ * 4, cudaMemcpyDeviceToHost), "read x");
}

void Runtime::read_last_topk(int32_t* out) {
    ck(cudaStreamSynchronize(s_gpu_), "sync");
    ck(cudaMemcpy(out, d_topk_, static_cast<size_t>(mu_) * K_ * 4, cudaMemcpyDeviceToHost), "read topk");
}

void Runtime::capture_router(int step) {
    if (step < 0 || step > max_steps_) throw std::invalid_argument("capture_router: step out of range");
    if (step && !h_cap_hn_) {
        const size_t rows = static_cast<size_t>(L_) * N_;
        ck(cudaHostAlloc(reinterpret_cast<void**>(&h_cap_hn_), rows * H_ * 2, 0), "cap_hn");
        ck(cudaHostAlloc(reinterpret_cast<void**>(&h_cap_topk_), rows * K_ * 4, 0), "cap_topk");
        ck(cudaHostAlloc(reinterpret_cast<void**>(&h_cap_topw_), rows * K_ * 4, 0), "cap_topw");
    }
    capture_step_ = step;
}

size_t Runtime::debug_read(const std::string& name, void* out, size_t cap) {
    const void* src = nullptr;
    size_t bytes = 0;
    if (name == "cap_hn" || name == "cap_topk" || name == "cap_topw") {  // router tap (host, pinned)
        const size_t rows = static_cast<size_t>(L_) * N_;
        src = name == "cap_hn" ? static_cast<const void*>(h_cap_hn_)
              : name == "cap_topk" ? static_cast<const void*>(h_cap_topk_) : static_cast<const void*>(h_cap_topw_);
        bytes = src ? rows * (name == "cap_hn" ? H_ * 2 : K_ * 4) : 0;
    } else if (name == "h") { src = d_h_; bytes = static_cast<size_t>(mu_) * H_ * 4; }
    else if (name == "hn") { src = d_hn_; bytes = static_cast<size_t>(mu_) * H_ * 2; }
    else if (name == "topk") { src = d_topk_; bytes = static_cast<size_t>(mu_) * K_ * 4; }
    else if (name == "topw") { src = d_topw_; bytes = static_cast<size_t>(mu_) * K_ * 4; }
    else if (name == "qkv_bf16") { src = d_qkv_bf16_ + static_cast<size_t>(M_ - 1) * mu_ * W_; bytes = static_cast<size_t>(mu_) * W_ * 2; }
    else if (name == "attn_in") { src = d_attn_in_ + static_cast<size_t>(M_ - 1) * Rmu_ * Ho_ * 2; bytes = static_cast<size_t>(Rmu_) * Ho_ * 2; }
    else if (name == "y") { src = d_y_; bytes = static_cast<size_t>(Re_) * H_ * 4; }
    else if (name == "inv") { src = d_inv_; bytes = static_cast<size_t>(mu_) * K_ * 4; }
    else if (name == "counts") { src = d_cnt_; bytes = static_cast<size_t>(E_) * 4; }
    else if (name == "offsets") { src = d_off_; bytes = static_cast<size_t>(E_ + 1) * 4; }
    else if (name == "logits") { src = d_logits_; bytes = static_cast<size_t>(mu_) * V_ * 4; }
    else if (name == "xe") { src = d_xe_; bytes = static_cast<size_t>(Re_) * H_ * 2; }
    else if (name == "inter") { src = d_inter_; bytes = static_cast<size_t>(Re_) * F_ * 2; }
    else if (name == "kcache" || name == "vcache") {  // host KV [L][N][nkv][max_ctx][d] (A_g = 0)
        src = name[0] == 'k' ? h_kcache_ : h_vcache_;
        bytes = src ? static_cast<size_t>(L_) * N_ * nkv_ * max_ctx_ * d_ * 2 : 0;
    } else if (name == "kpool" || name == "vpool") {  // paged device KV (A_g = 1)
        src = name[0] == 'k' ? d_kpool_ : d_vpool_;
        bytes = src ? static_cast<size_t>(L_) * N_ * max_pages_ * nkv_ * page_ * d_ * 2 : 0;
    }
    else throw std::invalid_argument("unknown debug buffer " + name);
    if (out) {
        if (cap < bytes) throw std::invalid_argument("debug_read: buffer too small");
        ck(cudaStreamSynchronize(s_gpu_), "sync");
        ck(cudaMemcpy(out, src, bytes, cudaMemcpyDefault), "debug read");
    }
    return bytes;
}

cudaEvent_t Runtime::take_event() {
    if (event_next_ == event_pool_.size()) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "event");
        event_pool_.push_back(e);
    }
    return event_pool_[event_next_++];
}

// Every kernel launch of a GPU task goes through kl(): error check, launch
// count, and a CUDA event recorded right after it on the compute stream.
// Consecutive events (the task's start event first) give the live per-kernel
// breakdown reported by decode() — no extra synchronisation.
void Runtime::kl(const char* name, cudaError_t e) {
    ck(e, name);
    ++launches_;
    static const bool sync_each = [] {  // diagnostic knob: MLT_SYNC_EACH=1 names the kernel that faults
        const char* v = std::getenv("MLT_SYNC_EACH");
        return v && v[0] == '1';
    }();
    if (sync_each) ck(cudaStreamSynchronize(s_gpu_), name);
    if (pdl_) return;  // no per-kernel events inside a PDL chain
    cudaEvent_t ev = take_event();
    ck(cudaEventRecord(ev, s_gpu_), "event");
    marks_.push_back({name, ev});
}

void Runtime::mark_start(cudaEvent_t task_start) { marks_.push_back({nullptr, task_start}); }

unsigned long long* Runtime::ktimer(const char* name) {
    if (static_cast<int>(ktime_names_.size()) >= ktime_cap_) return nullptr;
    ktime_names_.push_back(name);
    return d_ktime_ + 2 * (ktime_names_.size() - 1);
}

// Dense projections have few 128-row blocks (QKV 48, O 32 for 8x7B), too
// few to stream their weights over all SMs: split K so (row block x K-split)
// tiles cover the chip (each weight byte is still read once).  The fp32
// partials are reduced by the consumer (rope_qkv for QKV, the router kernel
// for O), in fixed order.  Tokens stay in one chunk (<= 256).
void Runtime::dense_tiling(int row_blocks, int& n_cap, int& n_chunks, int& k_splits) const {
    // the register-decode codec GEMM holds <= 64 tokens per chunk and runs 2 CTAs per SM
    n_cap = std::min(codec_mode_ == 2 ? 64 : 256, Rmu_);
    n_chunks = (mu_ + n_cap - 1) / n_cap;
    k_splits = std::max(1, std::min(kMaxSplits, gemm_slots() / (row_blocks * n_chunks)));
}

// Encoded-weight settings of a projection / expert GEMM (lm_head stays bf16):
// codec 1 = tcgen05 with in-smem decode (gemm_tc.cu), codec 2 = register
// decode + mma.sync (gemm_codec.cu: <= 64 tokens per chunk, <= 32 for gate/up),
// codec 3 = tcgen05 with A decoded into TMEM (gemm_tc.cu, decoupled rings).
void Runtime::codec_args(mltk::GemmArgs& a, int kind) const {
    a.codec = codec_mode_;
    if (codec_mode_ == 4) a.enc_tile = c4_tile_[kind];
    if (codec_mode_ == 2) a.n_cap = std::min(a.n_cap, a.n_mats == 2 ? 32 : 64);
    if (codec_mode_ >= 2) a.codec_raw = any_raw_ ? 1 : 0;  // raw fallback tiles need 16 KiB ring slots
}

// ---------------------------------------------------------------------------
// Task actions.  step/layer/mb are the 1-based fields of sim::Task.
// ---------------------------------------------------------------------------
namespace {
void kk(cudaError_t e, const char* what) { ck(e, what); }
}  // namespace

void Runtime::act_pre_attn(const Ctx& c, int step, int layer, int mb) {
    const int t0 = (mb - 1) * mu_;
    const int g = (step - 1) * L_ + layer;
    const int l = layer - 1;
    if (layer == 1) {
        const int32_t* src = (step == 1 || c.forced) ? d_tok_in_ + static_cast<size_t>(step - 1) * N_ + t0
                                                     : d_tok_out_ + static_cast<size_t>(step - 2) * N_ + t0;
        kl("embed", mltk::launch_embed(src, d_embed_, mu_, H_, d_x_ + static_cast<size_t>(t0) * H_, s_gpu_));
    }
    uint8_t* xn = d_xn_ + static_cast<size_t>(mb - 1) * Rmu_ * H_ * 2;
    if (layer == 1 || coll_)  // otherwise the previous layer's combine produced it
        kl("rmsnorm_pack", mltk::launch_rmsnorm_pack(d_x_ + static_cast<size_t>(t0) * H_, d_attn_norm_[l], mu_, H_,
                                                     ext_.rms_eps, xn, Rmu_, s_gpu_));
    mltk::GemmArgs a;
    a.a_table = dev_tables_ + (static_cast<size_t>(l) * 2 + slot_of(g)) * table_entries_ + tab_qkv_;
    a.n_mats = 1;
    a.G = 1;
    a.RB = W_ / 128;
    a.K = H_;
    a.b = xn;
    a.R = Rmu_;
    a.rows_dense = mu_;
    dense_tiling(W_ / 128, a.n_cap, a.n_chunks, a.k_splits);
    a.split_stride = static_cast<int64_t>(Rmu_) * W_;
    a.epi = mltk::kEpiF32;
    a.out_f32 = d_qkv_f32_;
    a.ldo = W_;
    a.timing = ktimer("qkv_gemm");
    codec_args(a, kWqkv);
    kl("qkv_gemm", mltk::launch_gemm(a, num_sms_, s_gpu_));
    const int32_t* pos = d_pos_ + static_cast<size_t>(step - 1) * N_ + t0;
    uint16_t* qkv = d_qkv_bf16_ + static_cast<size_t>(mb - 1) * mu_ * W_;
    mltk::KvAppend kv;  // A_g = 1: this step's k/v go straight into the paged pool
    if (policy_.attn_on_gpu) {
        kv.k_pool = d_kpool_;
        kv.v_pool = d_vpool_;
        kv.block_table = d_block_table_ + static_cast<size_t>(l) * N_ * max_pages_;
        kv.max_pages = max_pages_;
        kv.seq = d_seq_ + t0;
    }
    kl("rope_qkv", mltk::launch_rope_qkv(d_qkv_f32_, a.k_splits, a.split_stride, pos, d_rope_, mu_, nq_, nkv_,
                                         d_, qkv, s_gpu_, policy_.attn_on_gpu ? &kv : nullptr));
}

void Runtime::act_offload_qkv(int layer, int mb) {
    (void)layer;
    const size_t off = static_cast<size_t>(mb - 1) * mu_ * W_;
    kk(cudaMemcpyAsync(h_qkv_ + off, d_qkv_bf16_ + off, static_cast<size_t>(mu_) * W_ * 2, cudaMemcpyDeviceToHost,
                       s_d2h_),
       "offload qkv");
}

void Runtime::act_cpu_attn(int step, int layer, int mb) { host_attention(layer - 1, mb - 1, step); }

void Runtime::act_load_hidden(int layer, int mb) {
    (void)layer;
    const size_t off = static_cast<size_t>(mb - 1) * Rmu_ * Ho_ * 2;
    kk(cudaMemcpyAsync(d_attn_in_ + off, h_attn_ + off, static_cast<size_t>(Rmu_) * Ho_ * 2, cudaMemcpyHostToDevice,
                       s_h2d_),
       "load hidden");
}

void Runtime::act_gpu_attn(int step, int layer, int mb) {
    const int t0 = (mb - 1) * mu_;
    const int l = layer - 1;
    const uint16_t* qkv = d_qkv_bf16_ + static_cast<size_t>(mb - 1) * mu_ * W_;
    // this step's k/v were stored into the pool by rope_qkv (PreAttn)
    const int32_t* ctx = d_pos_ + static_cast<size_t>(max_steps_) * N_ + static_cast<size_t>(step - 1) * N_ + t0;
    const int32_t* bt = d_block_table_ + static_cast<size_t>(l) * N_ * max_pages_;
    // one CTA per (token, kv head), no split-KV: splitting a token's pages
    // over CTAs (mlt_gqa_decode_paged_split) measured slower at every decode
    // shape here (mu = 16/32/64, ctx 528: 18.9/20.5/56 vs 12.8/17.9/29.9 us,
    // profiles/r02_attention_split_kv.txt) — each short split CTA pays the
    // page-pipeline ramp and the partial merge
    kl("gqa_decode_paged", mltk::launch_gqa_decode_paged(qkv, W_, d_kpool_, d_vpool_, bt, max_pages_, d_seq_ + t0,
                                                         ctx, mu_, nq_, nkv_, d_, page_, d_attn_gpu_, Rmu_,
                                                         nullptr, s_gpu_));
}

void Runtime::act_post_attn(const Ctx& c, int step, int layer, int mb) {
    (void)c;
    const int t0 = (mb - 1) * mu_;
    const int g = (step - 1) * L_ + layer;
    const int l = layer - 1;
    const uint8_t** tab = dev_tables_ + (static_cast<size_t>(l) * 2 + slot_of(g)) * table_entries_;
    float* x = d_x_ + static_cast<size_t>(t0) * H_;
    uint8_t* xn = d_xn_ + static_cast<size_t>(mb - 1) * Rmu_ * H_ * 2;  // next layer's normed operand
    // O projection + residual
    mltk::GemmArgs o;
    o.a_table = tab + tab_o_;
    o.RB = H_ / 128;
    o.K = Ho_;  // this rank's heads (row-parallel O under TP)
    o.b = policy_.attn_on_gpu ? d_attn_gpu_ : d_attn_in_ + static_cast<size_t>(mb - 1) * Rmu_ * Ho_ * 2;
    o.R = Rmu_;
    o.rows_dense = mu_;
    dense_tiling(H_ / 128, o.n_cap, o.n_chunks, o.k_splits);
    const bool o_split = o.k_splits > 1;
    o.split_stride = static_cast<int64_t>(mu_) * H_;
    o.out_f32 = o_split ? d_hparts_ : d_h_;
    o.ldo = H_;
    o.residual = coll_ ? nullptr : x;  // unsplit single GPU: residual in the GEMM epilogue
    o.ldr = H_;
    o.timing = ktimer("o_gemm");
    codec_args(o, kWo);
    kl("o_gemm", mltk::launch_gemm(o, num_sms_, s_gpu_));
    if (coll_) {
        // TP all-reduce #1: h = x + sum over ranks of this rank's O partial
        if (o_split)
            kl("sum_parts", mltk::launch_sum_parts(d_hparts_, o.k_splits, o.split_stride, nullptr, d_h_,
                                                   static_cast<int64_t>(mu_) * H_, s_gpu_));
        coll_->all_reduce_sum(d_h_, static_cast<size_t>(mu_) * H_, s_gpu_);
        kl("router", mltk::launch_router(d_h_, d_ffn_norm_[l], ext_.rms_eps, nullptr, d_router_[l], mu_, H_, E_,
                                         K_, d_hn_, nullptr, d_topk_, d_topw_, s_gpu_, 1, 0, x, d_h_));
    } else {
        // (split-K reduce + residual ->) RMSNorm + router
        kl("router", mltk::launch_router(o_split ? d_hparts_ : d_h_, d_ffn_norm_[l], ext_.rms_eps, nullptr,
                                         d_router_[l], mu_, H_, E_, K_, d_hn_, nullptr, d_topk_, d_topw_, s_gpu_,
                                         o_split ? o.k_splits : 0, o.split_stride, o_split ? x : nullptr,
                                         o_split ? d_h_ : nullptr));
    }
    if (capture_step_ == step) {  // router tap: this layer's router input and choice (parity probe)
        const size_t row = static_cast<size_t>(l) * N_ + t0;
        kk(cudaMemcpyAsync(h_cap_hn_ + row * H_, d_hn_, static_cast<size_t>(mu_) * H_ * 2, cudaMemcpyDeviceToHost,
                           s_gpu_), "capture hn");
        kk(cudaMemcpyAsync(h_cap_topk_ + row * K_, d_topk_, static_cast<size_t>(mu_) * K_ * 4, cudaMemcpyDeviceToHost,
                           s_gpu_), "capture topk");
        kk(cudaMemcpyAsync(h_cap_topw_ + row * K_, d_topw_, static_cast<size_t>(mu_) * K_ * 4, cudaMemcpyDeviceToHost,
                           s_gpu_), "capture topw");
    }
    kl("moe_permute", mltk::launch_moe_permute(d_topk_, d_hn_, mu_, H_, E_, K_, d_cnt_, d_off_, d_perm_, d_inv_,
                                               d_xe_, Re_, s_gpu_));
    // experts: gate/up (SiLU fused) -> down -> combine
    mltk::GemmArgs gu;
    gu.a_table = tab + tab_w13_;
    gu.n_mats = 2;
    gu.G = E_;
    gu.RB = F_ / 128;
    gu.K = H_;
    gu.b = d_xe_;
    gu.R = Re_;
    gu.b_off = d_off_;
    gu.b_cnt = d_cnt_;
    gu.n_cap = ncap_e_;
    gu.epi = mltk::kEpiSiluPacked;
    gu.out_packed = d_inter_;
    gu.out_R = Re_;
    static const bool no_sk = [] {  // diagnostic knob: MLT_NO_STREAM_K=1 runs gate/up without the tail
        const char* e = std::getenv("MLT_NO_STREAM_K");
        return e && e[0] == '1';
    }();
    gu.sk_scratch = no_sk ? nullptr : d_sk_scratch_;
    gu.sk_count = d_sk_count_;
    gu.sk_rows = Rmu_;  // a token routes to an expert at most once: rows per group <= mu
    gu.timing = ktimer("expert_gateup_gemm");
    codec_args(gu, kW1);
    kl("expert_gateup_gemm", mltk::launch_gemm(gu, num_sms_, s_gpu_));
    mltk::GemmArgs dn;
    dn.a_table = tab + tab_w2_;
    dn.G = E_;
    dn.RB = H_ / 128;
    dn.K = F_;
    dn.b = d_inter_;
    dn.R = Re_;
    dn.b_off = d_off_;
    dn.b_cnt = d_cnt_;
    dn.n_cap = ncap_e_;
    dn.out_f32 = d_y_;
    dn.ldo = H_;
    dn.k_splits = down_splits_;
    dn.split_stride = static_cast<int64_t>(Re_) * H_;
    dn.timing = ktimer("expert_down_gemm");
    codec_args(dn, kW2);
    kl("expert_down_gemm", mltk::launch_gemm(dn, num_sms_, s_gpu_));
    if (coll_) {
        // TP all-reduce #2: x = h + sum over ranks of this rank's top-k combine (h2 shard)
        kl("moe_combine", mltk::launch_moe_combine(nullptr, d_y_, H_, d_inv_, d_topw_, mu_, H_, K_, d_cbuf_, s_gpu_,
                                                   nullptr, 0.f, nullptr, 0, down_splits_,
                                                   static_cast<int64_t>(Re_) * H_));
        coll_->all_reduce_sum(d_cbuf_, static_cast<size_t>(mu_) * H_, s_gpu_);
        kl("residual_add", mltk::launch_sum_parts(d_cbuf_, 1, 0, d_h_, x, static_cast<int64_t>(mu_) * H_, s_gpu_));
    } else {
        // + the next layer's attention norm (or the final norm) fused
        kl("moe_combine", mltk::launch_moe_combine(d_h_, d_y_, H_, d_inv_, d_topw_, mu_, H_, K_, x, s_gpu_,
                                                   layer == L_ ? d_final_norm_ : d_attn_norm_[l + 1],
                                                   ext_.rms_eps, xn, Rmu_, down_splits_,
                                                   static_cast<int64_t>(Re_) * H_));
    }
    if (layer == L_) {  // step epilogue: final norm -> lm_head -> greedy ids
        if (coll_)
            kl("rmsnorm_pack", mltk::launch_rmsnorm_pack(x, d_final_norm_, mu_, H_, ext_.rms_eps, xn, Rmu_, s_gpu_));
        mltk::GemmArgs lm;
        lm.a_table = d_lm_table_;
        lm.RB = V_ / 128;
        lm.K = H_;
        lm.b = xn;
        lm.R = Rmu_;
        lm.rows_dense = mu_;
        lm.n_cap = std::min(256, Rmu_);  // 250+ row blocks already fill the chip
        lm.n_chunks = (mu_ + lm.n_cap - 1) / lm.n_cap;
        lm.out_f32 = d_logits_;
        lm.ldo = V_;
        kl("lm_head_gemm", mltk::launch_gemm(lm, num_sms_, s_gpu_));
        kl("argmax", mltk::launch_argmax(d_logits_, mu_, V_, d_tok_out_ + static_cast<size_t>(step - 1) * N_ + t0,
                                         nullptr, s_gpu_));
    }
}

void Runtime::act_weight_to_gpu(int g, int page) {
    if (!layer_blob_bytes_) return;
    const int l = (g - 1) % L_;
    const auto [b, e] = page_range(page);
    if (e <= b) return;
    const uint8_t* src = opt_.pin_weights ? host_blob_ + static_cast<int64_t>(l) * layer_blob_bytes_
                                          : staging_ + static_cast<int64_t>(slot_of(g)) * layer_blob_bytes_;
    kk(cudaMemcpyAsync(dev_pool_ + static_cast<int64_t>(slot_of(g)) * layer_blob_bytes_ + b, src + b, e - b,
                       cudaMemcpyHostToDevice, s_h2d_),
       "weight page");
}

void Runtime::act_weight_to_pinned(int g, int page) {
    if (opt_.pin_weights || !layer_blob_bytes_) return;  // blob already page-locked
    const int l = (g - 1) % L_;
    const auto [b, e] = page_range(page);
    uint8_t* dst = staging_ + static_cast<int64_t>(slot_of(g)) * layer_blob_bytes_;
    const uint8_t* src = host_blob_ + static_cast<int64_t>(l) * layer_blob_bytes_;
    const int64_t chunk = 1 << 20;
#pragma omp parallel for schedule(static) num_threads(4)
    for (int64_t off = b; off < e; off += chunk) std::memcpy(dst + off, src + off, std::min(chunk, e - off));
}

}  // namespace mlt
