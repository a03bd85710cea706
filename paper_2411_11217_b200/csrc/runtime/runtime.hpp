// The B200 decode runtime: budget-capped device arena, paged weight store,
// host KV + host-core attention, and the CGOPipe executor.
//
// One Runtime per GPU.  It is the engine behind the reference's per-layer
// decode step: `decode()` builds the reference ScheduleDag for the policy
// (lightplan::sim::build_schedule, identical issue order) and EXECUTES it —
// GPU tasks on a compute stream, weight pages and hidden uploads on an H2D
// copy stream, QKV offloads on a D2H stream, CPU attention on host cores —
// returning the measured sim::Timeline (replacing sim::simulate,
// proj/src/pipesim.cpp:350-406) and a measured LatencyBreakdown.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "collective.hpp"
#include "exec_plan.hpp"
#include "host_gqa.hpp"
#include "lightplan/pipesim.hpp"
#include "lightplan/planner.hpp"

namespace mltk {
struct GemmArgs;
}

namespace mlt {

struct ModelExt {
    int vocab = 32000;
    float rms_eps = 1e-5f;
    float rope_theta = 1e6f;
    float lm_head_scale = 4.0f;
    uint64_t seed = 1234;
};

struct RuntimeOptions {
    int device = 0;
    double budget_bytes = 16e9;  // every runtime device allocation comes from this arena
    int max_ctx = 0;             // KV capacity per sequence
    int host_threads = 0;        // CPU attention threads (0: all)
    int pin_weights = 1;         // 1: streamed blob pinned; 0: pageable + pinned staging ring
    int exact_gates = 1;         // 1: data-exact weight gates; 0: reference gates (all pages of g)
    int tp_rank = 0, tp_size = 1;  // tensor parallelism (one process per GPU)
    uint8_t nccl_id[128] = {};     // ncclUniqueId from rank 0 (tp_size > 1)
    bool tp_shard_only = false;    // one shard alone on this GPU, all-reduce elided (measurement)
    int collective = 0;            // tp_size > 1: 0 NCCL, 1 host-staged shared memory (collective_host.cpp)
    // Caller-owned weights instead of the synthetic PRNG: get(ctx, layer,
    // kind, expert) returns the FULL row-major bf16 tensor (TensorKind;
    // layer -1 for embed / lm_head / final norm).  Used during construction only.
    const uint16_t* (*weight_fn)(void* ctx, int layer, int kind, int expert) = nullptr;
    void* weight_ctx = nullptr;
    bool weight_codec = false;     // store/stream/read projection + expert weights encoded (weight_codec.hpp)
    bool pdl = true;               // programmatic dependent launch on all-GPU (resident, A_g = 1) schedules
    int expert_down_splits = 0;    // 0: auto (codec: best last-wave fill in 1..8; raw: 1)
    int schedule = -1;             // -1: CGOPipe (S4 when A_g = 1); else a ScheduleKind to execute
    int prefill_chunk_tokens = 0;  // 0: largest prefill chunk the budget allows
};

// Throws std::invalid_argument unless every ids[i] is in [0, vocab).
void check_token_ids(const int32_t* ids, int64_t n, int vocab, const char* what);

// Bump allocator over one cudaMalloc of the budget (SURVEY.md §7 hard part 5).
class Arena {
  public:
    Arena(size_t bytes);
    ~Arena();
    void* alloc(size_t bytes, const char* what);
    size_t used() const { return used_; }
    size_t capacity() const { return cap_; }
    const std::string& log() const { return log_; }

  private:
    uint8_t* base_ = nullptr;
    size_t cap_ = 0, used_ = 0;
    std::string log_;
};

struct DecodeReport {
    double seconds = 0;              // wall time of the executed DAG (device clock)
    double tokens_per_second = 0;
    lightplan::LatencyBreakdown measured;  // per-layer means of the measured timeline
    double h2d_weight_bytes = 0;     // bytes of weight pages moved
    double h2d_bytes = 0, d2h_bytes = 0;
    double steady_layer_time = 0;
    double utilization[5] = {0, 0, 0, 0, 0};
    int gpu_launches = 0;
    std::string verify;              // verify_timeline_tol result on the measured timeline
    // Live per-launch timing of the dominant kernel pair (expert gate/up +
    // down GEMM of one micro-batch), CUDA events on the compute stream.
    double expert_ms_total = 0;
    int expert_launches = 0;
    double qkv_o_ms_total = 0;       // dense QKV + O projections (pairs per micro-batch-layer)
    int dense_launches = 0;
    struct KernelTime {
        std::string name;
        double ms = 0;
        int launches = 0;
    };
    std::vector<KernelTime> kernels;  // (empty: the event breakdown is Runtime::kernel_events(), on demand)
    std::vector<KernelTime> kernel_exec;  // in-kernel first-CTA-start to last-CTA-end (GEMMs)
};

// GPU prefill ("for the prefill stage, we perform all the
// computation on GPU and offload KV cache to CPU"; cost model planner.cpp:
// 110-150).  Device-timed with CUDA events around the whole call, host
// token upload and id download included.
struct PrefillReport {
    double seconds = 0;
    double tokens_per_second = 0;   // prompt tokens / s
    int64_t prompt_tokens = 0;
    int chunk_tokens = 0;           // token capacity of one chunk
    int chunks_per_layer = 0;
    double h2d_weight_bytes = 0, h2d_bytes = 0, d2h_bytes = 0;
    double gpu_busy_seconds = 0;    // sum over chunks of compute-stream time
    int gpu_launches = 0;
};

class Runtime {
  public:
    Runtime(const lightplan::ModelSpec& model, const ModelExt& ext, const lightplan::Policy& policy,
            const RuntimeOptions& opt);
    ~Runtime();
    Runtime(const Runtime&) = delete;
    Runtime& operator=(const Runtime&) = delete;

    // Synthetic prompt-stage KV for positions [0, prompt_len) of every
    // sequence (uniform(-1,1) bf16, oracle orc_fill_kv semantics); sets every
    // sequence's position to prompt_len.
    void prefill_synthetic(int prompt_len, uint64_t seed);
    void set_positions(const int32_t* pos);
    // GPU prefill of real prompts: tokens = the N prompts concatenated
    // (sequence i has lens[i] >= 1 tokens), first_ids[N] = the greedy token
    // after each prompt.  Zigzag order (layer by layer over chunks of whole
    // sequences); the residual stream of all prompt tokens lives in pinned
    // host memory between layers, KV goes to the host cache (A_g = 0) or the
    // paged device pool (A_g = 1).  Sets every position to lens[i].
    PrefillReport prefill(const int32_t* tokens, const int32_t* lens, int32_t* first_ids);
    const std::vector<int32_t>& positions() const { return pos_; }

    // `steps` decode steps for all N sequences.  tokens_in: [N] host ids of
    // step 0; forced: optional [steps][N] host ids (teacher forcing); out:
    // [steps][N] host greedy ids.  Host->device copy of the inputs and
    // device->host copy of the ids are inside the measured region.
    DecodeReport decode(const int32_t* tokens_in, const int32_t* forced, int steps, int32_t* out,
                        lightplan::sim::ScheduleDag* dag_out = nullptr,
                        lightplan::sim::Timeline* timeline_out = nullptr);
    // The same on a caller-built schedule: `dag` must be a build_schedule DAG
    // of this runtime's schedule kind, layers and micro-batches (checked);
    // the number of decode steps is the DAG's (forced/out are [steps][N]).
    DecodeReport execute(const lightplan::sim::ScheduleDag& dag, const int32_t* tokens_in, const int32_t* forced,
                         int32_t* out, lightplan::sim::ScheduleDag* dag_out = nullptr,
                         lightplan::sim::Timeline* timeline_out = nullptr);
    // The reference DAG this runtime executes for `steps` decode steps.
    lightplan::sim::ScheduleDag schedule(int steps) const;

    // Debug/test taps (device -> host copies, synchronous).
    void read_residual(float* host_out);          // x [N, H] fp32
    void read_last_topk(int32_t* host_idx);       // last micro-batch's topk [mu, K]
    size_t debug_read(const std::string& name, void* host_out, size_t cap);
    // Router tap: during decode step `step` (1-based, of the next decode()
    // call; 0 = off) every layer's router input hn (bf16 [N, H]), top-k ids
    // and weights are copied to host buffers on the compute stream (readable
    // via debug_read "cap_hn" [L][N][H] u16, "cap_topk" [L][N][K] i32,
    // "cap_topw" [L][N][K] f32).  A parity probe, off on measured paths.
    void capture_router(int step);

    double achieved_weight_ratio() const { return achieved_rw_; }
    int64_t streamed_bytes_per_layer() const { return layer_blob_bytes_; }
    size_t arena_used() const { return arena_->used(); }
    std::string arena_log() const { return arena_->log(); }
    const lightplan::Policy& policy() const { return policy_; }
    const lightplan::ModelSpec& model() const { return model_; }
    double pin_seconds() const { return pin_seconds_; }
    double gen_seconds() const { return gen_seconds_; }
    double bytes_per_weight() const {
        double bytes = 0, weights = 0;
        for (const auto& b : cat_.blocks) {
            bytes += static_cast<double>(b.bytes);
            weights += 128.0 * static_cast<double>(b.K);
        }
        return weights > 0 ? bytes / weights : 0.0;
    }
    int codec_mode() const { return codec_mode_; }
    std::vector<DecodeReport::KernelTime> kernel_events() const;  // last call's per-kernel event deltas
    int raw_blocks() const {
        int n = 0;
        for (const auto& b : cat_.blocks) n += b.raw ? 1 : 0;
        return n;
    }

    // --- task actions (called by the executor) ---
    struct Ctx;
    void act_pre_attn(const Ctx& c, int step, int layer, int mb);
    void act_offload_qkv(int layer, int mb);
    void act_cpu_attn(int step, int layer, int mb);
    void act_load_hidden(int layer, int mb);
    void act_post_attn(const Ctx& c, int step, int layer, int mb);
    void act_weight_to_gpu(int global_layer, int page);
    void act_weight_to_pinned(int global_layer, int page);
    void act_gpu_attn(int step, int layer, int mb);

    cudaStream_t stream(lightplan::sim::Resource r) const;
    int launches() const { return launches_; }

  private:
    DecodeReport run(lightplan::sim::ScheduleDag dag, const int32_t* tokens_in, const int32_t* forced, int steps,
                     int32_t* out, lightplan::sim::ScheduleDag* dag_out, lightplan::sim::Timeline* timeline_out);
    void build_catalog();
    // this rank's packed (SW128) rows of catalog block b of layer l
    void packed_block(int l, const WeightBlock& b, uint16_t* dst) const;
    // the first n elements of an unsharded tensor (router, norms, embedding)
    void plain_tensor(int l, int kind, int64_t n, float scale, bool is_norm, uint16_t* dst) const;
    const uint16_t* ext_tensor(int l, int kind, int expert) const;
    void scan_raw_blocks();  // codec + caller weights: blocks the code cannot hold -> raw_mask_
    void dense_tiling(int row_blocks, int& n_cap, int& n_chunks, int& k_splits) const;
    void codec_args(mltk::GemmArgs& a, int kind) const;  // kind: the GEMM's weight kind (kWqkv, kWo, kW1, kW2)
    // resident CTA slots of the weight GEMMs: 2 per SM for the register-decode codec GEMM
    int gemm_slots() const { return codec_mode_ == 2 ? 2 * num_sms_ : num_sms_; }
    int codec_mode_ = 0;   // 0 bf16 tiles, 1 encoded (tcgen05 path), 2 encoded fragment order (mma.sync)
    bool any_raw_ = false; // codec: some block is a raw fallback (tagged page-table entry)
    std::vector<uint8_t> raw_mask_;  // codec: per catalog block, stored raw (fallback)
    // codec 4: capacity (records + escapes per tile) and tile bytes per TensorKind,
    // sized by scan_raw_blocks from the weights
    int c4_cap_[16] = {44, 44, 44, 44, 44, 44, 44, 44, 44, 44, 44, 44, 44, 44, 44, 44};
    int c4_tile_[16] = {11600, 11600, 11600, 11600, 11600, 11600, 11600, 11600,
                        11600, 11600, 11600, 11600, 11600, 11600, 11600, 11600};
    static constexpr int kMaxSplits = 8;
    void allocate();
    void generate_weights();
    void host_attention(int layer, int mb, int step);
    int slot_of(int global_layer) const { return global_layer & 1; }
    // The schedule this runtime executes: opt_.schedule, or CGOPipe / S4 by A_g.
    lightplan::sim::ScheduleKind schedule_kind() const {
        using K = lightplan::sim::ScheduleKind;
        if (opt_.schedule < 0) return policy_.attn_on_gpu ? K::S4 : K::CgoPipe;
        const K k = static_cast<K>(opt_.schedule);
        if ((k == K::S4) != policy_.attn_on_gpu)
            throw lightplan::sim::UnsupportedCombinationError(std::string(lightplan::sim::to_string(k)) +
                                                              (policy_.attn_on_gpu ? " needs A_g = 0" : " needs A_g = 1"));
        return k;
    }
    std::pair<int64_t, int64_t> page_range(int page) const {  // [begin, end) within layer blob
        return mlt::page_range(layer_blob_bytes_, M_, page);
    }
    Catalog cat_;

    lightplan::ModelSpec model_;
    ModelExt ext_;
    lightplan::Policy policy_;
    RuntimeOptions opt_;
    // dims; under TP nq_, nkv_, F_, W_ and Ho_ (attention output width) are
    // this rank's shard (exec_plan.hpp Shard)
    int N_, mu_, M_, H_, F_, E_, K_, nq_, nkv_, d_, W_, V_, L_, Ho_;
    Shard shard_;
    ShardMap maps_[4];
    HostCores host_cores_;  // launcher / attention cores of the current decode
    std::unique_ptr<Collective> coll_;
    float* d_cbuf_ = nullptr;  // [mu, H] TP expert-combine partial (all-reduced)
    int Rmu_, Re_, ncap_, ncap_e_;
    int num_sms_ = 148;
    int down_splits_ = 1;  // K-splits of the expert down GEMM (partials in d_y_)

    std::unique_ptr<Arena> arena_;
    // weights
    int64_t layer_blob_bytes_ = 0, layer_res_bytes_ = 0;
    double achieved_rw_ = 0;
    uint8_t* host_blob_ = nullptr;     // [L][layer_blob_bytes_] (pinned or pageable)
    bool host_blob_pinned_ = false;
    uint8_t* staging_ = nullptr;       // pinned ring [2][layer_blob_bytes_] when !pin_weights
    uint8_t* dev_res_ = nullptr;       // [L][layer_res_bytes_]
    uint8_t* dev_pool_ = nullptr;      // [2][layer_blob_bytes_]
    const uint8_t** dev_tables_ = nullptr;  // [L][2 slots][table_entries]
    int table_entries_ = 0;
    int tab_qkv_ = 0, tab_o_ = 0, tab_w13_ = 0, tab_w2_ = 0;  // offsets within a table
    uint16_t *d_embed_ = nullptr, *d_lm_ = nullptr, *d_final_norm_ = nullptr;
    std::vector<uint16_t*> d_attn_norm_, d_ffn_norm_, d_router_;
    float2* d_rope_ = nullptr;
    const uint8_t** d_lm_table_ = nullptr;

    // activations
    float* d_x_ = nullptr;              // [N, H] residual
    uint16_t* d_qkv_bf16_ = nullptr;    // [M][mu][W]
    uint8_t* d_attn_in_ = nullptr;      // [M][Rmu*H] packed
    uint8_t* d_xn_ = nullptr;           // [Rmu*H] packed
    float* d_qkv_f32_ = nullptr;        // [kMaxSplits][Rmu, W] split-K partials
    float* d_h_ = nullptr;              // [mu, H]
    float* d_hparts_ = nullptr;         // [kMaxSplits][mu, H] O-projection split-K partials
    uint16_t* d_hn_ = nullptr;          // [mu, H]
    int32_t *d_topk_ = nullptr, *d_cnt_ = nullptr, *d_off_ = nullptr, *d_perm_ = nullptr, *d_inv_ = nullptr;
    float* d_topw_ = nullptr;
    uint8_t* d_xe_ = nullptr;           // [Re*H] packed
    uint8_t* d_inter_ = nullptr;        // [Re*F] packed
    float* d_y_ = nullptr;              // [Re, H]
    float* d_sk_scratch_ = nullptr;  // gate/up stream-K tail: fp32 parts [#SMs][2][Rmu][128]
    unsigned long long* d_sk_count_ = nullptr;  // [#SMs] 64-bit monotonic arrival counters
    float* d_logits_ = nullptr;         // [Rmu, V]
    int32_t* d_tok_in_ = nullptr;       // [max_steps][N]
    int32_t* d_tok_out_ = nullptr;      // [max_steps][N]
    int32_t* d_pos_ = nullptr;          // [max_steps][N]
    int32_t* d_seq_ = nullptr;          // [N]
    int max_steps_ = 256;  // decode steps per call (DBRX gen 128 runs in one call)
    // GPU attention (A_g = 1): paged KV pool
    uint16_t *d_kpool_ = nullptr, *d_vpool_ = nullptr;
    int32_t* d_block_table_ = nullptr;  // [L][N][max_pages]
    int max_pages_ = 0, page_ = 16;
    uint8_t* d_attn_gpu_ = nullptr;

    // host side
    uint16_t* h_qkv_ = nullptr;   // pinned [M][mu][W]
    uint8_t* h_attn_ = nullptr;   // pinned [M][Rmu*H]
    uint16_t* h_kcache_ = nullptr;  // [L][N][nkv][max_ctx][d]
    uint16_t* h_vcache_ = nullptr;
    int32_t* h_tok_ = nullptr;    // pinned [max_steps][N] in / out staging
    int capture_step_ = 0;        // router tap (capture_router)
    uint16_t* h_cap_hn_ = nullptr;
    int32_t* h_cap_topk_ = nullptr;
    float* h_cap_topw_ = nullptr;
    std::vector<int32_t> pos_;
    int max_ctx_ = 0;
    int cur_forced_ = 0, cur_steps_ = 0;
    std::vector<int32_t> step_pos_;  // [steps][N] positions used by the running decode

    cudaStream_t s_gpu_ = nullptr, s_h2d_ = nullptr, s_d2h_ = nullptr;
    int launches_ = 0;
    bool pdl_ = false;  // this decode runs its kernels as a PDL chain
    // per-kernel marks recorded by the GPU worker during decode(): (name,
    // event after the launch); name == nullptr marks a task's start event
    std::vector<std::pair<const char*, cudaEvent_t>> marks_;
    void kl(const char* name, cudaError_t launch_status);
    cudaEvent_t take_event();
    // in-kernel %globaltimer slots (GEMMs): true execution time without the
    // host-launch gaps that event deltas on an idle stream include
    unsigned long long* d_ktime_ = nullptr;
    std::vector<const char*> ktime_names_;
    int ktime_cap_ = 0;
    unsigned long long* ktimer(const char* name);

  public:
    void mark_start(cudaEvent_t task_start);

  private:
    // prefill scratch (allocated from the arena on first use) and host residual store
    void prefill_alloc(int64_t total_tokens, int max_len);
    int pf_T_ = 0;                       // chunk token capacity
    int pf_R_ = 0, pf_Re_ = 0;
    float* pf_x_[2] = {nullptr, nullptr};  // [T, H] fp32 residual, double-buffered
    uint8_t* pf_xn_ = nullptr;           // packed [R_T, H] (also the attention output)
    uint16_t* pf_qkv_ = nullptr;         // [T, W] roped bf16
    float* pf_h_ = nullptr;              // [T, H]
    uint16_t* pf_hn_ = nullptr;          // [T, H]
    int32_t *pf_topk_ = nullptr, *pf_perm_ = nullptr, *pf_inv_ = nullptr;
    float* pf_topw_ = nullptr;
    uint8_t* pf_xe_ = nullptr;           // packed [Re_T, H]
    uint8_t* pf_inter_ = nullptr;        // packed [Re_T, F]
    float* pf_y_ = nullptr;              // [Re_T, H] (also the QKV fp32 output)
    uint16_t* pf_kst_[2] = {nullptr, nullptr};  // K/V staging [2][T * nkv * d] per buffer
    int32_t* pf_meta_ = nullptr;         // per-chunk metadata (device)
    int64_t pf_meta_cap_ = 0;            // int32 entries
    float* h_pfx_ = nullptr;             // pinned [tokens][H] residual store
    int64_t h_pfx_tokens_ = 0;
    std::vector<cudaEvent_t> event_pool_;
    std::vector<cudaEvent_t> task_ev_;  // per-task start / end events of the executor, reused across calls
    void ensure_task_events(size_t n);
    void prefill_task_events(int steps);
    size_t event_next_ = 0;
    double pin_seconds_ = 0, gen_seconds_ = 0;

  public:
    struct Ctx {
        int steps;
        bool forced;
    };
};

}  // namespace mlt
