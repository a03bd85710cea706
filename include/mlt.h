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
/* estimate_throughput, planner.hpp:74-75 */
int mlt_estimate_throughput(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                            const mlt_workload_spec_t* workload, const mlt_policy_t* policy,
                            mlt_plan_result_t* out);

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

#ifdef __cplusplus
}
#endif

#endif /* MLT_H_ */
