/*
 * mlt.h — C ABI of the B200 MoE-Lightning decode hot path ("mlt" =
 * MoE-Lightning on Tensor cores).
 *
 * This is the drop-in boundary.  Every entry point is
 * extern "C", takes plain pointers and sizes, never throws, and returns an
 * int status (MLT_OK = 0, negative on error; mlt_last_error() gives a
 * thread-local message).  C++ exceptions of the reference API map onto the
 * status codes below:
 *   InfeasiblePolicyError       (planner.hpp:12-14)  -> MLT_ERR_INFEASIBLE
 *   UnsupportedCombinationError (pipesim.hpp:13-15)  -> MLT_ERR_UNSUPPORTED
 *   CycleDetectedError          (pipesim.hpp:16-18)  -> MLT_ERR_CYCLE
 *   EmptyTimelineError          (pipesim.hpp:19-21)  -> MLT_ERR_EMPTY
 *   std::invalid_argument                            -> MLT_ERR_INVALID
 *
 * The POD structs mirror the reference C++ structs field for field, in the
 * same order (bool -> int32_t).  Which reference interface each function
 * replaces is cited on the declaration.  INTEGRATION.md shows the ctypes /
 * C++ binding a reference maintainer would add.
 */
#ifndef MLT_H_
#define MLT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLT_OK 0
#define MLT_ERR_INVALID (-1)
#define MLT_ERR_INFEASIBLE (-2)
#define MLT_ERR_UNSUPPORTED (-3)
#define MLT_ERR_CYCLE (-4)
#define MLT_ERR_EMPTY (-5)
#define MLT_ERR_CUDA (-6)
#define MLT_ERR_BUDGET (-7)
#define MLT_ERR_INTERNAL (-8)
#define MLT_ERR_NO_FEASIBLE (-9) /* NoFeasiblePolicyError (planner.hpp:16-18) */

/* ---- spec structs: reference include/lightplan/config.hpp:12-56 ---------- */
typedef struct mlt_hardware_spec_t {
    double gpu_mem_bytes, cpu_mem_bytes, gpu_bw, cpu_bw, link_bw, gpu_flops, cpu_flops;
} mlt_hardware_spec_t;

typedef struct mlt_model_spec_t {
    int64_t layers, hidden_dim, ffn_dim, q_heads, kv_heads, experts, top_k;
    double weight_dtype_bytes, kv_dtype_bytes;
} mlt_model_spec_t;

typedef struct mlt_workload_spec_t {
    int64_t prompt_len, gen_len;
} mlt_workload_spec_t;

typedef struct mlt_policy_t {
    int64_t batch, micro_batch;
    int32_t attn_on_gpu, ffn_on_gpu;
    double weights_on_gpu, kv_on_gpu;
} mlt_policy_t;

/* ---- cost model: reference opcost.hpp:16-76 ------------------------------ */
typedef struct mlt_op_profile_t {
    double flops, gpu_bytes, cpu_bytes, link_bytes;
} mlt_op_profile_t;

typedef struct mlt_layer_weight_bytes_t {
    double experts, qkv, output, router;
} mlt_layer_weight_bytes_t;

typedef struct mlt_transfer_sizes_t {
    double qkv_offload, hidden_upload, weight_stream, kv_upload;
} mlt_transfer_sizes_t;

/* ---- planner: reference planner.hpp:25-69 -------------------------------- */
typedef struct mlt_latency_breakdown_t {
    double link_upload, gpu_attention, gpu_ffn, cpu_attention, cpu_ffn, layer_total;
} mlt_latency_breakdown_t;

typedef struct mlt_memory_footprint_t {
    double gpu_bytes, cpu_bytes;
    int32_t feasible;
} mlt_memory_footprint_t;

typedef struct mlt_plan_result_t {
    mlt_policy_t policy;
    mlt_latency_breakdown_t breakdown;
    mlt_memory_footprint_t memory;
    double decode_throughput, generation_throughput, objective;
} mlt_plan_result_t;

const char* mlt_last_error(void);
/* Status of the last failed call on this thread (for NULL-returning builders). */
int mlt_last_status(void);
const char* mlt_version(void);

/* ParsedConfig (config.hpp:89-94 of the reference). */
typedef struct mlt_config_t {
    mlt_hardware_spec_t hardware;
    mlt_model_spec_t model;
    mlt_workload_spec_t workload;
    mlt_policy_t policy;
    int32_t has_policy;
} mlt_config_t;

/* parse_config_text (config.hpp:116): INI text -> config.  MLT_OK, or
 * MLT_ERR_INVALID with *err_line = the 1-based line of a parse error (0: not
 * tied to a line, e.g. a missing section) or -1 for validation issues, and
 * the message (ConfigParseError::message / format_issues) in msg. */
int mlt_parse_config(const char* text, mlt_config_t* out, int32_t* err_line, char* msg, size_t msg_cap);
/* serialize_config (config.hpp:121): writes at most cap bytes (NUL-terminated)
 * and the full length to *len. */
int mlt_serialize_config(const mlt_config_t* config, char* buf, size_t cap, size_t* len);

/* validate(HardwareSpec/ModelSpec/WorkloadSpec/Policy), config.hpp:75-78.
 * Any pointer may be NULL (skipped).  Returns the number of issues (>= 0);
 * the formatted issue list (format_issues) is written to msg. */
int mlt_validate(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                 const mlt_workload_spec_t* workload, const mlt_policy_t* policy, char* msg,
                 size_t msg_cap);

/* attention_decode_profile / moe_ffn_profile / projection_profiles
 * (opcost.hpp:31-53). out[0]=attention, out[1]=ffn, out[2]=qkv, out[3]=o. */
int mlt_op_profiles(const mlt_model_spec_t* model, double tokens, double ctx, double weights_on_gpu,
                    mlt_op_profile_t out[4]);
/* layer_weight_bytes, opcost.hpp:55-65 */
int mlt_layer_weight_bytes(const mlt_model_spec_t* model, mlt_layer_weight_bytes_t* out);
/* transfer_sizes, opcost.hpp:67-74 */
int mlt_transfer_sizes(const mlt_model_spec_t* model, const mlt_policy_t* policy, double ctx,
                       mlt_transfer_sizes_t* out);
/* memory_totals, opcost.hpp:76; out[0]=weight_bytes, out[1]=kv_cache_bytes */
int mlt_memory_totals(const mlt_model_spec_t* model, const mlt_workload_spec_t* workload,
                      int64_t batch, double out[2]);

/* layer_latency, planner.hpp:43-44 (MLT_ERR_INFEASIBLE when it does not fit) */
int mlt_layer_latency(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                      const mlt_workload_spec_t* workload, const mlt_policy_t* policy, double ctx,
                      mlt_latency_breakdown_t* out);
/* memory_footprint, planner.hpp:55-56 */
int mlt_memory_footprint(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                         const mlt_workload_spec_t* workload, const mlt_policy_t* policy,
                         mlt_memory_footprint_t* out);
/* apply_tensor_parallelism, planner.hpp:58-60.  b200_rule != 0 selects the
 * B200 deviation: link_bw := min(tp * link_bw, host_read_cap). */
int mlt_apply_tensor_parallelism(const mlt_hardware_spec_t* hw, int tp, int b200_rule,
                                 double host_read_cap, mlt_hardware_spec_t* out);
/* B200 HRM of a tp-way group: estimate_throughput on the TP-scaled spec
 * (mlt_apply_tensor_parallelism with the B200 rule) plus the NVLink roof of
 * the two fp32 all-reduces per layer per micro-batch (ring bytes
 * 2(tp-1)/tp x mu*h1*4 at nvlink_bw B/s per direction) added to every
 * layer's GPU FFN term (lightplan::estimate_throughput_b200). */
int mlt_estimate_throughput_b200(const mlt_hardware_spec_t* tp_hw, const mlt_model_spec_t* model,
                                 const mlt_workload_spec_t* workload, const mlt_policy_t* policy,
                                 int tp, double nvlink_bw, mlt_plan_result_t* out);
/* estimate_throughput, planner.hpp:74-75 */
int mlt_estimate_throughput(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                            const mlt_workload_spec_t* workload, const mlt_policy_t* policy,
                            mlt_plan_result_t* out);

/* ---- hierarchical roofline: reference hrm.hpp:13-74 ---------------------- */
#define MLT_LEVEL_GPU 0 /* MemoryLevel::Gpu */
#define MLT_LEVEL_CPU 1 /* MemoryLevel::Cpu */
/* attainable_local, hrm.hpp:17 (level: MLT_LEVEL_*) */
int mlt_hrm_attainable_local(int level, double intensity, const mlt_hardware_spec_t* hw, double* out);
/* attainable_cross, hrm.hpp:22 */
int mlt_hrm_attainable_cross(double gpu_intensity, double cpu_intensity, const mlt_hardware_spec_t* hw,
                             double* out);
/* turning_point_p1 / turning_point_p2, hrm.hpp:26-30 */
int mlt_hrm_turning_point_p1(double cpu_intensity, const mlt_hardware_spec_t* hw, double* out);
int mlt_hrm_turning_point_p2(double gpu_intensity, const mlt_hardware_spec_t* hw, double* out);
/* balance_gap, hrm.hpp:34 */
int mlt_hrm_balance_gap(double gpu_intensity, double cpu_intensity, const mlt_hardware_spec_t* hw,
                        double* out);
/* RooflineGrid, hrm.hpp:57-61 */
typedef struct mlt_roofline_grid_t {
    double min_intensity, max_intensity;
    int32_t points_per_decade;
} mlt_roofline_grid_t;
/* roofline_csv(roofline_series(profiles, names, hw, grid)), hrm.hpp:66-73.
 * grid NULL = the defaults.  Writes at most cap bytes (NUL-terminated) and
 * the full length to *len; MLT_ERR_INVALID on empty input (std::invalid_argument). */
int mlt_roofline_csv(const mlt_op_profile_t* profiles, const char* const* names, int n,
                     const mlt_hardware_spec_t* hw, const mlt_roofline_grid_t* grid, char* buf, size_t cap,
                     size_t* len);

/* ---- policy search: reference planner.hpp:77-116 ------------------------- */
typedef struct mlt_search_grid_t {
    const int64_t* micro_batch_values;
    int32_t n_micro_batch_values;
    const int64_t* micro_batch_counts;
    int32_t n_micro_batch_counts;
    const double* weight_ratio_values;
    int32_t n_weight_ratio_values;
    const double* kv_ratio_values;
    int32_t n_kv_ratio_values;
    const int32_t* attn_on_gpu_values;
    int32_t n_attn_on_gpu_values;
    const int32_t* ffn_on_gpu_values;
    int32_t n_ffn_on_gpu_values;
} mlt_search_grid_t;

/* search_policy (planner.hpp:110-116); grid NULL = SearchGrid::defaults();
 * objective 0 = tokens/s, 1 = layer latency; ctx_override < 0 = s + n/2.
 * MLT_ERR_NO_FEASIBLE when nothing fits (message names the constraint). */
int mlt_search_policy(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                      const mlt_workload_spec_t* workload, const mlt_search_grid_t* grid,
                      int objective, double ctx_override, mlt_plan_result_t* out);
/* SearchGrid::candidate_count (grid NULL = defaults). */
int64_t mlt_search_candidate_count(const mlt_search_grid_t* grid);

/* ---- batcher: reference batcher.hpp:10-40 (Algorithm 2) ------------------ */
typedef struct mlt_batch_params_t {
    int64_t n_ub, ubs, gen_len, cache_size;
    int32_t flush_partials;
} mlt_batch_params_t;

/* batch_requests: returns the number of micro-batches; out_batch[i] = the
 * micro-batch of request i (-1 = aborted), out_slot[i] = its position there
 * (for aborted requests: the abort order); -2 = left in an unsealed
 * partition (only with flush_partials = 0, batcher.hpp:24-27). */
int mlt_batch_requests(const char* const* ids, const int64_t* input_len, int32_t n,
                       const mlt_batch_params_t* params, int32_t* out_batch, int32_t* out_slot);

/* ---- CGOPipe scheduler: reference pipesim.hpp:23-136 --------------------- */
enum { MLT_SCHED_CGOPIPE = 0, MLT_SCHED_S2 = 1, MLT_SCHED_S3 = 2, MLT_SCHED_S4 = 3 };
enum {
    MLT_TASK_PRE_ATTN = 0, MLT_TASK_OFFLOAD_QKV, MLT_TASK_CPU_ATTN, MLT_TASK_LOAD_HIDDEN,
    MLT_TASK_POST_ATTN, MLT_TASK_WEIGHT_TO_PINNED, MLT_TASK_WEIGHT_TO_GPU, MLT_TASK_KV_LOAD,
    MLT_TASK_GPU_ATTN
};
enum { MLT_RES_GPU = 0, MLT_RES_CPU, MLT_RES_H2D, MLT_RES_D2H, MLT_RES_CTOPIN };

typedef struct mlt_step_durations_t {
    double pre_attn, offload_qkv, cpu_attn, load_hidden, post_attn, weight_stage, weight_upload,
        kv_load, gpu_attn;
} mlt_step_durations_t;

typedef struct mlt_task_t {
    int32_t kind, step, layer, microbatch, page, resource;
    double duration;
    int32_t n_deps;
} mlt_task_t;

typedef struct mlt_timeline_entry_t {
    int32_t task;
    double start, end;
} mlt_timeline_entry_t;

typedef struct mlt_sim_metrics_t {
    double makespan;
    double utilization[5];
    double steady_layer_time;
} mlt_sim_metrics_t;

typedef struct mlt_dag mlt_dag;

/* build_schedule(hw, model, workload, policy, kind, layers, steps),
 * pipesim.hpp:92-96.  Returns NULL on error (see mlt_last_error). */
mlt_dag* mlt_schedule_build(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                            const mlt_workload_spec_t* workload, const mlt_policy_t* policy,
                            int kind, int layers, int steps);
/* build_schedule(DurationProvider, ...) with a per-step duration table
 * durations[steps] (pipesim.hpp:85-86). */
mlt_dag* mlt_schedule_build_durations(const mlt_step_durations_t* durations, int kind, int layers,
                                      int steps, int micro_batches);
/* Build a DAG from raw task arrays (tests: malformed graphs). deps_flat holds
 * tasks[i].n_deps indices per task, concatenated. */
mlt_dag* mlt_dag_from_tasks(const mlt_task_t* tasks, int n_tasks, const int32_t* deps_flat,
                            int layers, int steps, int micro_batches, int kind);
void mlt_dag_free(mlt_dag* dag);
int mlt_dag_size(const mlt_dag* dag);
int mlt_dag_task(const mlt_dag* dag, int index, mlt_task_t* out, int32_t* deps, int deps_cap);
/* Canonical one-line-per-task text (%.17g durations, deps) used by the
 * schedule parity test.  Returns the needed length (excl. NUL). */
int mlt_dag_dump(const mlt_dag* dag, char* buf, size_t cap);
/* simulate, pipesim.hpp:114; entries must hold mlt_dag_size() items. */
int mlt_simulate(const mlt_dag* dag, mlt_timeline_entry_t* entries, double* makespan,
                 double busy[5]);
/* metrics, pipesim.hpp:126 */
int mlt_metrics(const mlt_dag* dag, const mlt_timeline_entry_t* entries, int n, double makespan,
                const double busy[5], mlt_sim_metrics_t* out);
/* verify_timeline, pipesim.hpp:131 (tol = 1e-9 reproduces the reference).
 * Returns MLT_OK when clean, 1 when violated (message in msg). */
int mlt_verify_timeline(const mlt_dag* dag, const mlt_timeline_entry_t* entries, int n,
                        double makespan, const double busy[5], double tol, char* msg,
                        size_t msg_cap);
/* timeline_json, pipesim.hpp:134-135.  Returns needed length. */
int mlt_timeline_json(const mlt_dag* dag, const mlt_timeline_entry_t* entries, int n,
                      double makespan, const double busy[5], const char* manifest_json,
                      char* buf, size_t cap);


/* ==== Kernel-level entry points (device pointers, caller-owned) ==========
 * Every pointer below is a device pointer unless named host_*; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  These are the hot-path
 * kernels of SURVEY.md §2c; the runtime (below) strings them together.  The
 * packed operand layout is defined in DESIGN.md §3 (kernels/common.cuh).
 */

/* Host: row-major bf16 [M, K] -> packed weight blocks (M % 128 == 0,
 * K % 64 == 0); dst holds M*K bf16. */
int mlt_pack_weight(const uint16_t* host_src, int64_t M, int64_t K, uint16_t* host_dst);
/* Lossless weight-tile codec: encode a packed [M, K] matrix
 * (M/128 row blocks x K/64 tiles of 16 KiB) into M/128*K/64 tiles of
 * mlt_codec_tile_bytes() = 12432 B each, same order (row block r starts at
 * r*(K/64)*12432).  MLT_ERR_INVALID if a tile's high bytes do not fit the
 * code (> 31 escapes). */
int mlt_codec_encode(const uint8_t* host_packed, int64_t M, int64_t K, uint8_t* host_out);
int mlt_codec_decode(const uint8_t* host_enc, int64_t tiles, uint8_t* host_packed);
int mlt_codec_tile_bytes(void);
/* The fragment-order code of the register-decode GEMM (GemmArgs codec = 2,
 * kernels/gemm_codec.cu; runtime/weight_codec.hpp frag_from_packed): encode a
 * packed [M, K] matrix row block by row block.  A row block with a tile the
 * code cannot hold is stored raw instead (K/64 tiles of 16 KiB in fragment
 * order) when raw_blocks (uint8[M/128], set to 1 for such blocks) is given;
 * without it that is MLT_ERR_INVALID.  Row block r starts at the sum of the
 * previous blocks' sizes.  Returns the number of raw blocks (>= 0). */
int mlt_codec_encode_frag(const uint8_t* host_packed, int64_t M, int64_t K, uint8_t* host_out,
                          uint8_t* raw_blocks);
/* The row-plane code of the TMEM-operand GEMM (GemmArgs codec = 3, kernels/
 * gemm_tc.cu; runtime/weight_codec.hpp rows_from_packed): same contract as
 * mlt_codec_encode_frag; raw fallback blocks are plain 16 KiB packed tiles. */
int mlt_codec_encode_rows(const uint8_t* host_packed, int64_t M, int64_t K, uint8_t* host_out,
                          uint8_t* raw_blocks);
/* The 3-bit row-plane code (GemmArgs codec = 4; runtime/weight_codec.hpp
 * codec4_encode_rows_tile): 11 stored bits per weight, mlt_codec4_tile_bytes()
 * = 11600 B per 64-k tile (7 tile-wide high bytes + a per-row slot with a
 * per-unit second value, a per-tile exponent phase, <= 44 records + escapes
 * per tile); same contract as
 * mlt_codec_encode_rows.  mlt_codec4_decode_rows is the host reference
 * decoder (encoded tiles -> 16 KiB packed tiles). */
int mlt_codec4_encode_rows(const uint8_t* host_packed, int64_t M, int64_t K, uint8_t* host_out,
                           uint8_t* raw_blocks);
int mlt_codec4_decode_rows(const uint8_t* host_enc, int64_t tiles, uint8_t* host_packed);
int mlt_codec4_tile_bytes(void);
/* Capacity variants: cap records + escapes per tile (<= 200), tiles of
 * mlt_codec4_tile_bytes_for(cap) = 11424 + 4 cap rounded up to 16 bytes (the
 * runtime sizes cap per weight kind); decode_rows_cap reads such tiles. */
int mlt_codec4_encode_rows_cap(const uint8_t* host_packed, int64_t M, int64_t K, int32_t cap, uint8_t* host_out,
                               uint8_t* raw_blocks);
int mlt_codec4_decode_rows_cap(const uint8_t* host_enc, int64_t tiles, int32_t cap, uint8_t* host_packed);
int mlt_codec4_tile_bytes_for(int32_t cap);
/* 16 KiB packed tiles -> fragment-order bf16 tiles (raw codec-2 blocks). */
int mlt_frag_pack(const uint8_t* host_packed, int64_t tiles, uint8_t* host_out);
/* Host-core GQA decode attention (A_g = 0: the CpuAttn task, pipesim.hpp:26,
 * PAPER.md:390-392/553; cost model cpu_attention, planner.cpp:42-44) — the
 * runtime's CpuAttn kernel on caller buffers.  q [T][nq][d] bf16 (roped);
 * kc, vc [T][nkv][max_ctx][d] bf16 (one contiguous stream per sequence and
 * kv head); ctx[t] in [1, max_ctx] valid rows; out [T][nq][d] bf16.  d must
 * be 128, nq % nkv == 0, nq / nkv <= 16.  threads <= 0: all host cores. */
int mlt_host_gqa_decode(const uint16_t* host_q, const uint16_t* host_k, const uint16_t* host_v,
                        const int32_t* host_ctx, int T, int nq, int nkv, int d, int max_ctx,
                        uint16_t* host_out, int threads);
/* Select the host GQA path process-wide: enable != 0 -> the AMX tile path
 * when the CPU has AMX-BF16 and the OS grants the tile state, else the
 * AVX-512 path.  Returns 1 if AMX is in use afterwards, 0 otherwise (never
 * an error).  Default: AMX when available (env MLT_HOST_AMX=0 disables). */
int mlt_host_gqa_use_amx(int enable);
/* Host: packed activation rows (capacity R) -> row-major bf16 [rows, K]. */
int mlt_unpack_rows(const uint8_t* host_packed, int64_t R, int64_t rows, int64_t K,
                    uint16_t* host_dst);
/* Host: row-major bf16 [rows, K] -> packed activation layout (capacity R). */
int mlt_pack_rows_host(const uint16_t* host_src, int64_t rows, int64_t K, int64_t R,
                       uint8_t* host_dst);

typedef struct mlt_gemm_args_t {
    const void* a_table; /* device array of const void*, [n_mats][G][RB] weight row blocks */
    int32_t n_mats, G, RB, K;
    const void* b;       /* packed activations, capacity R rows */
    int32_t R;
    const int32_t* b_off; /* [G+1] padded group row offsets or NULL (dense) */
    const int32_t* b_cnt; /* [G] rows per group or NULL (dense) */
    int32_t rows_dense, n_cap;
    int32_t epi;          /* 0: fp32 rows (+ residual); 1: silu(A0)*A1 -> packed bf16 */
    float alpha;
    float* out_f32;
    int32_t ldo;
    const float* residual;
    int32_t ldr;
    void* out_packed;
    int32_t out_R;
    int32_t n_chunks;     /* token chunks per (group, row block) spread over CTAs; 0 -> 1 */
    int32_t k_splits;     /* split-K: partial s written at out_f32 + s*split_stride; 0 -> 1 */
    int64_t split_stride; /* floats between partial outputs (residual ignored when split) */
    unsigned long long* trace; /* optional [gridDim][8] %globaltimer phase stamps per CTA
                                  (entry, setup done, first weight copy issued, first stage
                                  full, last MMA issued, first accumulator ready, epilogue
                                  done, exit) — a diagnostic, NULL in production */
    int32_t codec;             /* 1: every A row block is encoded (12432 B per 64-k tile, see
                                  mlt_codec_encode), expanded in smem by decoder warps (tcgen05);
                                  2: fragment-order encoded blocks (mlt_codec_encode_frag), decoded
                                  in registers and multiplied with mma.sync (n_cap <= 64, <= 32
                                  for n_mats = 2; kernels/gemm_codec.cu);
                                  3: row-plane encoded blocks (mlt_codec_encode_rows), each decoder
                                  thread expands one weight row into tensor memory and the
                                  tcgen05.mma reads A from TMEM (raw fallback blocks: tag bit 0);
                                  4: the same engine on 3-bit row-plane blocks
                                  (mlt_codec4_encode_rows, 11600 B per tile) */
    unsigned long long* ktrace; /* optional CTA-0 pipeline trace [4][256] %globaltimer stamps per
                                   k-block: producer issue, decoder start, decoder done, MMA start;
                                   codec 3: [6][256] per weight tile: producer issue, landed,
                                   decoded, TMEM slot granted, stored, MMA start */
    float* sk_scratch;         /* optional stream-K tail for epi = 1 (n_chunks = k_splits = 1): fp32
                                  scratch [#SMs][2][sk_rows][128]; NULL disables it */
    int64_t* sk_count;         /* [#SMs] 64-bit arrival counters, zeroed once by the caller */
    int32_t sk_rows;           /* row capacity per group for the scratch (>= max rows of a group) */
    int32_t dec_groups;        /* codec 1: decoder groups of 4 warps (2; 0 -> the default) */
    int32_t codec_raw;         /* codec 2: 1 when a page-table entry may carry tag bit 0 (a raw
                                  fragment-order block, mlt_codec_encode_frag raw_blocks) */
    int32_t enc_tile;          /* codec 4: bytes per encoded tile (mlt_codec4_tile_bytes_for(cap));
                                  0 -> 11600 (the default capacity, mlt_codec4_encode_rows) */
} mlt_gemm_args_t;

/* Grouped swap-AB tcgen05 GEMM (SURVEY.md §2c expert_gateup_silu /
 * expert_down / dense projections). */
int mlt_gemm(const mlt_gemm_args_t* args, void* stream);

int mlt_embed(const int32_t* tokens, const uint16_t* table, int T, int H, float* x_out,
              void* stream);
int mlt_rmsnorm_pack(const float* x, const uint16_t* gamma, int T, int H, float eps,
                     void* out_packed, int R, void* stream);
int mlt_pack_rows(const uint16_t* src, int ld, int T, int K, void* dst, int R, void* stream);
int mlt_rope_qkv(const float* qkv, const int32_t* pos, const void* rope_cos_sin, int T, int nq,
                 int nkv, int d, uint16_t* out, void* stream);

/* Router: top-k over the fixed-tree fp32 logits (bit-exact vs the oracle on
 * identical bf16 inputs).  Either x+gamma (fused RMSNorm) or hn_in. */
int mlt_router_topk(const float* x, const uint16_t* gamma, float eps, const uint16_t* hn_in,
                    const uint16_t* w_router, int T, int H, int E, int K, uint16_t* hn_out,
                    float* logits, int32_t* topk_idx, float* topk_w, void* stream);
/* Stable permutation + gather into the packed expert operand. */
int mlt_moe_permute(const int32_t* topk_idx, const uint16_t* hn, int T, int H, int E, int K,
                    int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv,
                    void* x_packed, int R, void* stream);
int mlt_moe_combine(const float* h, const float* y, int ldy, const int32_t* inv,
                    const float* topk_w, int T, int H, int K, float* x_out, void* stream);

/* Expert FFN of one MoE layer on the permuted operand: fused gate/up GEMM
 * (SiLU gating in the TMEM epilogue) -> down GEMM -> top-k weighted combine
 * with the residual h.  w13_table: [2][E][F/128] row blocks (W1 then W3);
 * w2_table: [E][H/128]; inter_packed capacity R rows of F; y fp32 [R, H]. */
int mlt_expert_ffn(const void* x_packed, int R, const int32_t* counts, const int32_t* offsets,
                   const void* w13_table, const void* w2_table, int E, int H, int F, int n_cap,
                   void* inter_packed, float* y, const int32_t* inv, const float* topk_w,
                   const float* h, int T, int K, float* x_out, void* stream);

int mlt_argmax(const float* logits, int T, int V, int32_t* ids, float* margin, void* stream);

int mlt_gqa_decode_paged(const uint16_t* q, int ldq, const uint16_t* k_pool,
                         const uint16_t* v_pool, const int32_t* block_table, int max_pages,
                         const int32_t* seq, const int32_t* ctx, int T, int nq, int nkv, int d,
                         int page, void* out_packed, int R, float* out_rowmajor, void* stream);
/* Split-KV variant: each (token, kv head)'s pages are split over `splits`
 * CTAs (0 = auto: the count in 1..max_splits that best fills whole waves of
 * SMs); scratch >= T*nq*max_splits*130 floats; counters >= T*nkv int32,
 * zeroed once by the caller (every launch leaves them zero).  Same output. */
int mlt_gqa_decode_paged_split(const uint16_t* q, int ldq, const uint16_t* k_pool, const uint16_t* v_pool,
                               const int32_t* block_table, int max_pages, const int32_t* seq,
                               const int32_t* ctx, int T, int nq, int nkv, int d, int page, void* out_packed,
                               int R, float* out_rowmajor, int splits, int max_splits, float* scratch,
                               int32_t* counters, void* stream);
/* Stream-K variant (gqa_decode_flat_kernel): `ctas` resident CTAs (0 = 2 per
 * SM) split the flattened (token, kv head, page) space evenly, partial
 * softmax states of shared (token, head) segments merged in warp order by the
 * last arriver.  scratch >= ctas*4*2*(nq/nkv)*130 floats; counters >= T*nkv
 * int32 zeroed once (left zero).  T <= 4096.  Same output. */
int mlt_gqa_decode_paged_flat(const uint16_t* q, int ldq, const uint16_t* k_pool, const uint16_t* v_pool,
                              const int32_t* block_table, int max_pages, const int32_t* seq, const int32_t* ctx, int T,
                              int nq, int nkv, int d, int page, void* out_packed, int R, float* out_rowmajor, int ctas,
                              float* scratch, int32_t* counters, void* stream);
int mlt_kv_append(const uint16_t* qkv_bf16, int nq, int nkv, int d, const int32_t* seq,
                  const int32_t* pos, int T, const int32_t* block_table, int max_pages, int page,
                  uint16_t* k_pool, uint16_t* v_pool, void* stream);

/* Causal GQA prefill attention (kernels/attention_prefill.cu).  qkv: roped
 * bf16 rows [T][W], W = (nq + 2 nkv) d; tiles: n_tiles x {first row of the
 * sequence, its length, first query position (multiple of 16), 0}; output
 * packed bf16 rows (capacity R) of width nq*d.  d = 128, nq/nkv <= 8. */
int mlt_prefill_attention(const uint16_t* qkv, int W, const int32_t* tiles, int n_tiles, int nq, int nkv,
                          int d, void* out_packed, int R, void* stream);
/* K/V rows of a prefill chunk -> per-sequence [nkv][len][d] staging (the
 * layout one strided copy lands in the host KV cache).  tok_seq/tok_pos per
 * row; seq_row0/seq_len per sequence of the chunk. */
int mlt_kv_stage(const uint16_t* qkv, int W, int nq, int nkv, int d, const int32_t* tok_seq,
                 const int32_t* tok_pos, const int32_t* seq_row0, const int32_t* seq_len, int T,
                 uint16_t* stage_k, uint16_t* stage_v, void* stream);

/* Host: rotary cos/sin table [max_pos][d/2] as (cos, sin) float pairs, angle
 * computed in double (theta^(-2i/d) * pos). */
int mlt_rope_table(int max_pos, int d, double theta, float* host_out);

/* Host link measurement (the b_cg of the B200 HardwareSpec): page-locked
 * host buffer (THP + cudaHostRegister, as the weight store) <-> device,
 * `bytes` per copy, best of `reps`, CUDA events.  out[0] = H2D GB/s,
 * out[1] = D2H GB/s, out[2] = H2D GB/s with a concurrent D2H stream. */
int mlt_measure_link(int device, size_t bytes, int reps, double out[3]);
/* Host DRAM bandwidth (the b_c of the HardwareSpec), all host threads:
 * out[0] = read GB/s (sum over `bytes`), out[1] = copy GB/s. */
int mlt_measure_host_bw(size_t bytes, double out[2]);

/* Host: synthetic weights, element i of tensor tid: splitmix64 counter PRNG
 * (DESIGN.md §3), bf16 RNE.  Multi-threaded. */
int mlt_synth_bf16(uint64_t seed, uint64_t tid, int64_t n, float scale, int is_norm,
                   uint16_t* host_out);

/* ==== Decode runtime (one per GPU) =======================================
 * The engine behind the reference's per-layer decode step: owns the
 * budget-capped device arena (every device allocation, SURVEY.md §7 hard
 * part 5), the pinned host weight store and HBM page pool, the host KV cache
 * and host-core attention, and the CGOPipe executor.  mlt_runtime_decode
 * builds the reference ScheduleDag for the policy (build_schedule,
 * pipesim.hpp:85-96), executes it on streams/threads, and returns the
 * measured per-layer breakdown (LatencyBreakdown fields, planner.hpp:25-35).
 * Thread-compatible: one caller per runtime.
 */
typedef struct mlt_runtime_options_t {
    int32_t device;
    double budget_bytes;   /* device memory cap for all runtime allocations */
    int32_t max_ctx;       /* KV capacity per sequence (>= s + n) */
    int32_t host_threads;  /* CPU attention threads, 0 = all */
    int32_t pin_weights;   /* 1: streamed weights page-locked; 0: pageable + pinned staging ring */
    int32_t vocab;
    float rms_eps, rope_theta, lm_head_scale;
    uint64_t seed;         /* synthetic-weight seed */
    int32_t exact_gates;   /* 1: data-exact weight gates (default); 0: reference gates,
                              every GPU task of layer g waits for all pages of g
                              (pipesim.cpp:131-148) */
    int32_t tp_rank, tp_size; /* tensor parallelism, one process per GPU (tp_size 0/1: off):
                                 heads + expert h2 sharded, 2 all-reduces per layer */
    uint8_t nccl_id[128];     /* mlt_nccl_unique_id() of rank 0, identical on every rank */
    int32_t schedule;         /* -1: CGOPipe (S4 when A_g = 1); else an mlt_schedule_build
                                 kind (0 CGOPipe, 1 S2, 2 S3, 3 S4; pipesim.hpp:20-21) to
                                 execute a baseline schedule on the same kernels */
    int32_t prefill_chunk_tokens; /* 0: largest chunk the budget allows (<= 8192 tokens) */
    int32_t tp_shard_only;    /* 1 (with tp_size > 1): run rank tp_rank's shard ALONE on this GPU
                                 with the all-reduce elided — a per-GPU throughput measurement
                                 of a tp_size job on one device (values are partial sums) */
    int32_t weight_codec;     /* 1: projection + expert weights are stored, paged and read by the
                                 GEMMs as encoded tiles (lossless, 24 % fewer bytes over PCIe and
                                 from HBM; mlt_codec_encode); numerics unchanged bit for bit */
    int32_t disable_pdl;      /* 1: no programmatic dependent launch (all-GPU schedules use it by
                                 default; per-kernel CUDA-event breakdowns need it off) */
    int32_t collective;       /* tp_size > 1: 0 = NCCL (nccl_id = ncclUniqueId); 1 = host-staged
                                 all-reduce through POSIX shared memory (ranks on one host, any
                                 number per GPU; nccl_id = a NUL-terminated rendezvous name,
                                 identical on every rank and unique per job) */
    int32_t expert_down_splits; /* K-splits of the expert down GEMM (fp32 partials summed in part
                                 order by the combine): 0 = auto (with weight_codec, the split
                                 in 1..8 that best fills the last wave of SMs; 1 without), else
                                 explicit; results are bit-identical for equal splits */
} mlt_runtime_options_t;

/* ncclUniqueId for a tensor-parallel group (call on rank 0, broadcast). */
int mlt_nccl_unique_id(uint8_t out[128]);

/* Tensor-parallel shard of one rank (GPU-free): local head / h2 counts and
 * the global rows / columns each local weight matrix covers. */
typedef struct mlt_tp_shard_t {
    int64_t q_heads, kv_heads, ffn, qkv_rows, o_k;
    int64_t ffn_off; /* first global h2 row of this rank's slice (128-row blocks, as even as
                        blocks allow: DBRX h2=10752 at tp=8 -> 1408 or 1280 rows) */
} mlt_tp_shard_t;
int mlt_tp_shard(const mlt_model_spec_t* model, int rank, int size, mlt_tp_shard_t* out);
/* Host: this rank's local weight matrix `kind` (5 wqkv, 6 wo, 8 w1, 9 w3,
 * 10 w2) of (layer, expert), row-major bf16 [rows, cols] exactly as the
 * runtime generates it (packed, then unpacked here for inspection). */
int mlt_synth_tp_weight(const mlt_model_spec_t* model, int rank, int size, uint64_t seed,
                        int layer, int kind, int expert, uint16_t* host_out, int64_t* rows,
                        int64_t* cols);

typedef struct mlt_decode_report_t {
    double seconds, tokens_per_second;
    mlt_latency_breakdown_t measured; /* per-layer means of the measured timeline */
    double h2d_weight_bytes, h2d_bytes, d2h_bytes, steady_layer_time;
    double utilization[5];
    int32_t gpu_launches;
    int32_t timeline_ok; /* 1 when verify_timeline passes on the measured timeline */
    /* live CUDA-event timing of the dominant kernels inside the decode */
    double expert_ms_total;  /* expert gate/up + down GEMM pairs */
    int32_t expert_launches;
    double dense_ms_total;   /* QKV and O projection GEMMs */
    int32_t dense_launches;
} mlt_decode_report_t;

typedef struct mlt_runtime_info_t {
    double achieved_weight_ratio;   /* realised r_w */
    double streamed_bytes_per_layer;
    double arena_used, arena_capacity;
    double pin_seconds, gen_seconds;
    double bytes_per_weight;  /* projection + expert weights as stored (2 = bf16; codec ~1.41 / 1.52) */
    double raw_blocks;        /* codec: 128-row blocks per layer stored raw (per-block fallback) */
    double codec_engine;      /* 0 bf16 tiles; 4 the 11-bit code (default), 3 the 12-bit code
                                 (MLT_CODEC_MODE=3 or the fallback), 1 / 2 the other engines */
} mlt_runtime_info_t;

typedef struct mlt_runtime mlt_runtime;

mlt_runtime* mlt_runtime_create(const mlt_model_spec_t* model, const mlt_policy_t* policy,
                                const mlt_runtime_options_t* options);
void mlt_runtime_destroy(mlt_runtime* rt);
/* Caller-owned weights instead of the synthetic ones (e.g. a real checkpoint).
 * get(ctx, layer, kind, expert) returns the FULL (unsharded) tensor as
 * row-major bf16 bits; layer = -1 for the model-level tensors.  kind:
 *   0 embed [vocab][h1]      1 lm_head [vocab][h1]   2 final_norm [h1]
 *   3 attn_norm [h1]         4 ffn_norm [h1]         5 wqkv [(n_q+2n_kv)d][h1]
 *     (q heads, then k heads, then v heads)          6 wo [h1][n_q d]
 *   7 router [n_e][h1]       8 w1 [h2][h1]  9 w3 [h2][h1]  10 w2 [h1][h2]
 * (expert = 0 for non-expert tensors).  Called only during this call, from
 * the calling thread; pointers need not outlive it; NULL = MLT_ERR_INVALID.
 * With weight_codec, row blocks the code cannot hold are stored raw (per-block
 * fallback, see mlt_runtime_info raw_blocks). */
typedef const uint16_t* (*mlt_weight_fn)(void* ctx, int layer, int kind, int expert);
mlt_runtime* mlt_runtime_create_with_weights(const mlt_model_spec_t* model, const mlt_policy_t* policy,
                                             const mlt_runtime_options_t* options, mlt_weight_fn get, void* ctx);
int mlt_runtime_info(const mlt_runtime* rt, mlt_runtime_info_t* out);
/* Synthetic prompt-stage KV for positions [0, prompt_len); positions := prompt_len. */
int mlt_runtime_prefill_synthetic(mlt_runtime* rt, int prompt_len, uint64_t seed);
/* GPU prefill of real prompts (cost
 * model planner.cpp:110-150).  tokens: the N prompts concatenated, lens[N]
 * >= 1 each (< max_ctx); first_ids[N]: the greedy token after each prompt.
 * Zigzag order (layer by layer over chunks of whole sequences, streamed
 * weights double-buffered in the HBM pool); KV to the host cache (A_g = 0)
 * or the paged device pool (A_g = 1).  Positions become lens[i]; decode
 * continues from there.  MLT_ERR_BUDGET when the arena has no room for a
 * chunk holding the longest prompt. */
typedef struct mlt_prefill_report_t {
    double seconds;              /* device-timed, host token upload and id download included */
    double tokens_per_second;    /* prompt tokens / s */
    int64_t prompt_tokens;
    int32_t chunk_tokens, chunks_per_layer;
    double h2d_weight_bytes, h2d_bytes, d2h_bytes;
    double gpu_busy_seconds;     /* compute-stream time summed over chunks */
    int32_t gpu_launches;
} mlt_prefill_report_t;
int mlt_runtime_prefill(mlt_runtime* r, const int32_t* tokens, const int32_t* lens, int32_t* first_ids,
                        mlt_prefill_report_t* rep);

int mlt_runtime_set_positions(mlt_runtime* rt, const int32_t* host_pos);
/* `steps` decode steps: host_tokens [N] (step-0 ids), host_forced [steps][N]
 * or NULL (teacher forcing), host_out [steps][N] greedy ids. */
int mlt_runtime_decode(mlt_runtime* rt, const int32_t* host_tokens, const int32_t* host_forced,
                       int steps, int32_t* host_out, mlt_decode_report_t* report);
/* sim::execute (lightplan/runtime.hpp; replaces sim::simulate, reference
 * pipesim.hpp:114): run a caller-built schedule — a build_schedule DAG
 * (mlt_schedule_build*) of this runtime's kind, layers and micro-batches —
 * instead of the runtime's own.  Decode steps = the DAG's step count;
 * host_forced / host_out are [steps][N].  MLT_ERR_INVALID for a DAG that does
 * not match the runtime, MLT_ERR_CYCLE for a cyclic one. */
int mlt_runtime_execute(mlt_runtime* rt, const mlt_dag* dag, const int32_t* host_tokens,
                        const int32_t* host_forced, int32_t* host_out, mlt_decode_report_t* report);
/* The graph the executor runs for `reference` (a build_schedule DAG of this
 * model/policy): same tasks and issue order; with exact_gates the
 * all-pages weight gates (pipesim.cpp:131-148) are replaced by the pages a
 * task actually reads; buffer-reuse (write-after-read) edges of the two-slot
 * page pool / staging ring are added to deps.  GPU-free; NULL on error.
 * info (optional) receives the realised residency split. */
mlt_dag* mlt_execution_dag(const mlt_dag* reference, const mlt_model_spec_t* model,
                           const mlt_policy_t* policy, int exact_gates,
                           mlt_runtime_info_t* info);
/* Live per-kernel breakdown of the last decode: JSON {"events": [...],
 * "exec": [...]} of {"name","ms","launches"}; "events" are CUDA-event deltas
 * on the compute stream (include host-launch gaps), "exec" the GEMMs'
 * in-kernel first-CTA-start..last-CTA-end time.  Returns length. */
int mlt_runtime_kernel_profile(mlt_runtime* rt, char* buf, size_t cap);
/* timeline_json of the last decode's measured timeline; returns length. */
int mlt_runtime_timeline_json(mlt_runtime* rt, char* buf, size_t cap);
int mlt_runtime_read_residual(mlt_runtime* rt, float* host_out);
/* Test tap: copy a named device buffer of the last micro-batch ("h", "hn",
 * "topk", "topw", "qkv_bf16", "attn_in", "y", "inv", "counts", "offsets",
 * "logits") to host; returns the byte count (host_out may be NULL). */
int mlt_runtime_debug_read(mlt_runtime* rt, const char* name, void* host_out, size_t cap);
/* Parity probe: arm a router tap for decode step `step` (1-based) of the next
 * mlt_runtime_decode call (0 = off).  Every layer's router input (bf16
 * [N, h1]) and top-k choice are then readable with mlt_runtime_debug_read
 * names "cap_hn" ([L][N][h1] u16), "cap_topk" ([L][N][k] i32), "cap_topw"
 * ([L][N][k] f32), so a caller can re-run the CPU router on identical inputs
 * at every layer (BASELINE: router top-k bit-exact). */
int mlt_runtime_capture_router(mlt_runtime* rt, int step);

#ifdef __cplusplus
}
#endif

#endif /* MLT_H_ */
