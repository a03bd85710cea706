// CGOPipe executor: runs a lightplan ScheduleDag on real resources and
// returns the measured Timeline (it replaces sim::simulate,
// proj/src/pipesim.cpp:350-406, with the same FIFO-per-resource semantics,
// proj/include/lightplan/pipesim.hpp:110-113).
//
// One launcher thread per resource walks that resource's tasks in issue
// order (SURVEY.md §7 hard part 1: enqueue in dependency-ready order, the
// event_oracle.cpp:22-53 loop with "enqueued" in place of "done"):
//   gpu  -> kernels on the compute stream      h2d -> cudaMemcpyAsync, copy engine
//   d2h  -> cudaMemcpyAsync, the other engine  cpu -> host attention (OpenMP)
//   ctopin -> DRAM -> pinned staging memcpy (only when weights are not pinned)
// A dependency on a device task is a cudaStreamWaitEvent on its end event
// (after the producer thread has recorded it); a host task waiting on a
// device task synchronises that event; anything waiting on a host task
// waits for its completion flag.  Device tasks are bracketed by CUDA events
// and host tasks by steady_clock, aligned on one reference event, so the
// measured timeline can be fed to metrics()/verify_timeline().
//
// The reference DAG does not encode buffer reuse (its model assumes the
// double buffer of planner.cpp:91-92 just works).  The executor adds the
// write-after-read edges that make reuse safe by construction: pages of
// global layer g+2 are uploaded into the pool slot of layer g only after
// every GPU task of layer g; staging pages likewise wait for the upload that
// read them.  simulate() on the augmented graph proves it acyclic first.
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../capi/status.hpp"
#include "host_layout.hpp"
#include "runtime.hpp"
#include "../kernels/kernels.hpp"

namespace mlt {

using lightplan::sim::Resource;
using lightplan::sim::ScheduleDag;
using lightplan::sim::Task;
using lightplan::sim::TaskKind;
using lightplan::sim::Timeline;

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void check_token_ids(const int32_t* ids, int64_t n, int vocab, const char* what) {
    if (!ids) throw std::invalid_argument(std::string(what) + ": null");
    for (int64_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= vocab)
            throw std::invalid_argument(std::string(what) + "[" + std::to_string(i) + "] = " + std::to_string(ids[i]) +
                                        " is not a token id in [0, " + std::to_string(vocab) + ")");
}

namespace {

bool on_device(Resource r) {
    return r == Resource::Gpu || r == Resource::HostToDevice || r == Resource::DeviceToHost;
}

struct Flags {
    std::mutex m;
    std::condition_variable cv;
    std::vector<char> ready;  // device: end event recorded; host: finished
    bool failed = false;
    std::string error;

    void set(int i) {
        {
            std::lock_guard<std::mutex> g(m);
            ready[i] = 1;
        }
        cv.notify_all();
    }
    void fail(const std::string& e) {
        {
            std::lock_guard<std::mutex> g(m);
            if (!failed) error = e;
            failed = true;
        }
        cv.notify_all();
    }
    bool wait(int i) {
        std::unique_lock<std::mutex> g(m);
        cv.wait(g, [&] { return ready[i] || failed; });
        return !failed;
    }
};

}  // namespace

// The reference DAG (lightplan::sim::build_schedule, pipesim.cpp:294-348) of
// this runtime's schedule kind for `steps` decode steps.  Durations are
// placeholders: the executor runs in issue order and dependency order only
// (the weight-upload estimate uses the page bytes at a nominal PCIe rate; it
// orders nothing).
// Per-kernel event deltas of the last decode call on the compute stream
// (diagnostic breakdown, mlt_runtime_kernel_profile "events"): read on demand
// after the call instead of inside it (tens of thousands of event queries
// were ~0.1 s of every decode call); valid until the next decode call.
std::vector<DecodeReport::KernelTime> Runtime::kernel_events() const {
    std::vector<DecodeReport::KernelTime> out;
    for (size_t k = 1; k < marks_.size(); ++k) {
        const char* name = marks_[k].first;
        if (!name) continue;  // a task start: the interval before it is not a kernel
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, marks_[k - 1].second, marks_[k].second), "elapsed");
        auto it = std::find_if(out.begin(), out.end(),
                               [&](const DecodeReport::KernelTime& kt) { return kt.name == name; });
        if (it == out.end()) {
            out.push_back({name, 0.0, 0});
            it = out.end() - 1;
        }
        it->ms += ms;
        it->launches += 1;
    }
    return out;
}

void Runtime::ensure_task_events(size_t n) {
    while (task_ev_.size() < n) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "event");
        task_ev_.push_back(e);
    }
}

void Runtime::prefill_task_events(int steps) {
    const ScheduleDag dag = schedule(std::max(1, std::min(steps, max_steps_)));
    size_t dev = 0;
    for (const Task& t : dag.tasks) dev += on_device(t.resource) ? 1 : 0;
    ensure_task_events(2 * dev);
}

ScheduleDag Runtime::schedule(int steps) const {
    const double link = 55e9;  // nominal; measured durations replace every modeled one
    return lightplan::sim::build_schedule(
        [&](int) {
            lightplan::sim::StepDurations d;
            d.pre_attn = d.post_attn = d.cpu_attn = d.gpu_attn = 1e-4;
            d.offload_qkv = d.load_hidden = d.kv_load = 1e-5;
            d.weight_upload = static_cast<double>(layer_blob_bytes_) / link;
            d.weight_stage = opt_.pin_weights ? 0.0 : static_cast<double>(layer_blob_bytes_) / link;
            return d;
        },
        schedule_kind(), L_, steps, M_);
}

DecodeReport Runtime::decode(const int32_t* tokens_in, const int32_t* forced, int steps, int32_t* out,
                             ScheduleDag* dag_out, Timeline* tl_out) {
    if (steps < 1 || steps > max_steps_)
        throw std::invalid_argument("steps must be in [1, " + std::to_string(max_steps_) + "]");
    return run(schedule(steps), tokens_in, forced, steps, out, dag_out, tl_out);
}

DecodeReport Runtime::execute(const ScheduleDag& dag, const int32_t* tokens_in, const int32_t* forced, int32_t* out,
                              ScheduleDag* dag_out, Timeline* tl_out) {
    // A caller-built DAG must describe THIS runtime's decode: tasks of its
    // schedule kind over its layers, micro-batches and pages; the step count
    // is the DAG's.
    using lightplan::sim::TaskKind;
    if (dag.tasks.empty()) throw lightplan::sim::EmptyTimelineError("execute: empty schedule");
    int steps = 0;
    for (const Task& t : dag.tasks) {
        steps = std::max(steps, t.step);
        const bool gpu_attn = t.kind == TaskKind::GpuAttn || t.kind == TaskKind::KvLoad;
        const bool host_attn = t.kind == TaskKind::CpuAttn || t.kind == TaskKind::OffloadQkv ||
                               t.kind == TaskKind::LoadHidden;
        if (t.step < 1 || t.layer < 1 || t.layer > L_ || t.microbatch < 0 || t.microbatch > M_ || t.page < 0 ||
            t.page > M_ || (gpu_attn && !policy_.attn_on_gpu) || (host_attn && policy_.attn_on_gpu))
            throw std::invalid_argument("execute: the schedule does not match this runtime's model/policy "
                                        "(build it with build_schedule for the same layers, micro-batches and A_g)");
    }
    if (steps > max_steps_)
        throw std::invalid_argument("execute: at most " + std::to_string(max_steps_) + " decode steps per call");
    lightplan::sim::simulate(dag);  // acyclic (CycleDetectedError otherwise)
    return run(dag, tokens_in, forced, steps, out, dag_out, tl_out);
}

DecodeReport Runtime::run(ScheduleDag dag, const int32_t* tokens_in, const int32_t* forced, int steps, int32_t* out,
                          ScheduleDag* dag_out, Timeline* tl_out) {
    const auto call_t0 = std::chrono::steady_clock::now();  // MLT_HOST_TIMING=1: host phases to stderr
    for (int i = 0; i < N_; ++i)
        if (pos_[i] + steps > max_ctx_) throw std::invalid_argument("KV capacity exceeded (max_ctx)");
    // token ids index the [vocab, h1] embedding on the device: reject bad ids here
    check_token_ids(tokens_in, N_, V_, "tokens_in");
    if (forced) check_token_ids(forced, static_cast<int64_t>(steps) * N_, V_, "forced");
    const int n = static_cast<int>(dag.tasks.size());
    if (opt_.exact_gates) apply_exact_gates(dag, cat_, M_);
    const auto extra = reuse_edges(dag);
    {
        ScheduleDag check = dag;  // prove the augmented graph acyclic
        for (int i = 0; i < n; ++i)
            check.tasks[i].deps.insert(check.tasks[i].deps.end(), extra[i].begin(), extra[i].end());
        lightplan::sim::simulate(check);
    }

    // ---- inputs (inside the measured region) ----
    step_pos_.assign(static_cast<size_t>(steps) * N_, 0);
    std::vector<int32_t> ctx(static_cast<size_t>(steps) * N_);
    for (int s = 0; s < steps; ++s)
        for (int i = 0; i < N_; ++i) {
            step_pos_[static_cast<size_t>(s) * N_ + i] = pos_[i] + s;
            ctx[static_cast<size_t>(s) * N_ + i] = pos_[i] + s + 1;
        }
    // All-GPU schedules (weights + KV resident, attention on the GPU) are
    // launch-bound chains of kernels on one stream: launch them with PDL so a
    // kernel's launch and setup (and its first weight tiles, prefetched to L2)
    // overlap its predecessor's tail.  Per-kernel events would serialise the
    // chain, so the per-kernel breakdown is taken without PDL (pdl_ false).
    pdl_ = opt_.pdl && policy_.attn_on_gpu && cat_.blob_bytes == 0;
    mltk::set_pdl(pdl_);
    struct PdlOff {
        ~PdlOff() { mltk::set_pdl(false); }
    } pdl_off;
    // task events come from the runtime's pool (pre-created for a 32-step
    // decode at construction, grown on demand, reused across calls): creating
    // tens of thousands per call was ~0.1 s of host work inside every decode
    std::vector<cudaEvent_t> ev_start(n, nullptr), ev_end(n, nullptr);
    {
        size_t dev = 0;
        for (int i = 0; i < n; ++i) dev += on_device(dag.tasks[i].resource) ? 1 : 0;
        ensure_task_events(2 * dev);
        size_t j = 0;
        for (int i = 0; i < n; ++i)
            if (on_device(dag.tasks[i].resource)) {
                ev_start[i] = task_ev_[j++];
                ev_end[i] = task_ev_[j++];
            }
    }
    cudaEvent_t e0, e_end;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e_end), "event");
    ck(cudaEventRecord(e0, s_gpu_), "event");
    ck(cudaEventSynchronize(e0), "event sync");
    const auto host_t0 = std::chrono::steady_clock::now();
    const double setup_s = std::chrono::duration<double>(host_t0 - call_t0).count();
    std::memcpy(h_tok_, tokens_in, N_ * 4);
    if (forced) std::memcpy(h_tok_, forced, static_cast<size_t>(steps) * N_ * 4);
    std::memcpy(h_tok_ + static_cast<size_t>(max_steps_) * N_, step_pos_.data(), step_pos_.size() * 4);
    std::memcpy(h_tok_ + static_cast<size_t>(max_steps_) * N_ * 2, ctx.data(), ctx.size() * 4);
    ck(cudaMemcpyAsync(d_tok_in_, h_tok_, static_cast<size_t>(forced ? steps : 1) * N_ * 4, cudaMemcpyHostToDevice,
                       s_gpu_),
       "tokens h2d");
    ck(cudaMemcpyAsync(d_pos_, h_tok_ + static_cast<size_t>(max_steps_) * N_, step_pos_.size() * 4,
                       cudaMemcpyHostToDevice, s_gpu_),
       "pos h2d");
    ck(cudaMemcpyAsync(d_pos_ + static_cast<size_t>(max_steps_) * N_, h_tok_ + static_cast<size_t>(max_steps_) * N_ * 2,
                       ctx.size() * 4, cudaMemcpyHostToDevice, s_gpu_),
       "ctx h2d");
    cudaEvent_t e_inputs;
    ck(cudaEventCreateWithFlags(&e_inputs, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(e_inputs, s_gpu_), "event");
    ck(cudaStreamWaitEvent(s_h2d_, e_inputs, 0), "wait");
    ck(cudaStreamWaitEvent(s_d2h_, e_inputs, 0), "wait");

    // ---- execute ----
    std::vector<double> h_start(n, 0), h_end(n, 0);
    Flags flags;
    flags.ready.assign(n, 0);
    const Ctx cctx{steps, forced != nullptr};
    cur_steps_ = steps;
    launches_ = 0;
    marks_.clear();
    event_next_ = 0;
    ktime_names_.clear();
    ck(cudaMemsetAsync(d_ktime_, 0xFF, static_cast<size_t>(ktime_cap_) * 16, s_gpu_), "timer reset");

    std::array<std::vector<int>, lightplan::sim::kResourceCount> fifo;
    for (int i = 0; i < n; ++i) fifo[static_cast<int>(dag.tasks[i].resource)].push_back(i);

    host_cores_ = host_cores(shard_.rank, opt_.tp_shard_only ? 1 : shard_.size);
    auto worker = [&](Resource r) {
        try {
            if (r != Resource::Cpu) pin_thread(host_cores_.launch);
            const cudaStream_t st = stream(r);
            ck(cudaSetDevice(opt_.device), "set device");
            for (int i : fifo[static_cast<int>(r)]) {
                const Task& t = dag.tasks[i];
                auto wait_dep = [&](int d) {
                    if (!flags.wait(d)) throw std::runtime_error("aborted");
                    const Resource rd = dag.tasks[d].resource;
                    if (on_device(rd)) {
                        if (on_device(r)) {
                            if (rd != r) ck(cudaStreamWaitEvent(st, ev_end[d], 0), "stream wait");
                        } else {
                            ck(cudaEventSynchronize(ev_end[d]), "event sync");
                        }
                    }
                };
                for (int d : t.deps) wait_dep(d);
                for (int d : extra[i]) wait_dep(d);
                if (on_device(r)) {
                    ck(cudaEventRecord(ev_start[i], st), "record");
                    if (r == Resource::Gpu) mark_start(ev_start[i]);
                    switch (t.kind) {
                        case TaskKind::PreAttn: act_pre_attn(cctx, t.step, t.layer, t.microbatch); break;
                        case TaskKind::PostAttn: act_post_attn(cctx, t.step, t.layer, t.microbatch); break;
                        case TaskKind::GpuAttn: act_gpu_attn(t.step, t.layer, t.microbatch); break;
                        case TaskKind::OffloadQkv: act_offload_qkv(t.layer, t.microbatch); break;
                        case TaskKind::LoadHidden: act_load_hidden(t.layer, t.microbatch); break;
                        case TaskKind::WeightToGpu: act_weight_to_gpu((t.step - 1) * L_ + t.layer, t.page); break;
                        case TaskKind::KvLoad: break;  // r_c = 1: KV resident, nothing to move
                        default: throw std::logic_error("host task on a device resource");
                    }
                    ck(cudaEventRecord(ev_end[i], st), "record");
                } else {
                    h_start[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - host_t0).count();
                    if (t.kind == TaskKind::CpuAttn) act_cpu_attn(t.step, t.layer, t.microbatch);
                    else if (t.kind == TaskKind::WeightToPinned)
                        act_weight_to_pinned((t.step - 1) * L_ + t.layer, t.page);
                    h_end[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - host_t0).count();
                }
                flags.set(i);
            }
        } catch (const std::exception& e) {
            flags.fail(e.what());
        }
    };
    {
        std::vector<std::thread> th;
        for (int r = 0; r < lightplan::sim::kResourceCount; ++r)
            if (!fifo[r].empty()) th.emplace_back(worker, static_cast<Resource>(r));
        for (auto& t : th) t.join();
    }
    if (flags.failed) {
        cudaDeviceSynchronize();
        for (int i = 0; i < n; ++i) {
            if (ev_start[i]) cudaEventDestroy(ev_start[i]);
            if (ev_end[i]) cudaEventDestroy(ev_end[i]);
        }
        throw std::runtime_error("executor: " + flags.error);
    }
    // join all streams into the compute stream, fetch the greedy ids
    for (cudaStream_t s : {s_h2d_, s_d2h_}) {
        cudaEvent_t j;
        ck(cudaEventCreateWithFlags(&j, cudaEventDisableTiming), "event");
        ck(cudaEventRecord(j, s), "record");
        ck(cudaStreamWaitEvent(s_gpu_, j, 0), "wait");
        cudaEventDestroy(j);
    }
    ck(cudaMemcpyAsync(h_tok_ + static_cast<size_t>(max_steps_) * N_ * 3, d_tok_out_, static_cast<size_t>(steps) * N_ * 4,
                       cudaMemcpyDeviceToHost, s_gpu_),
       "ids d2h");
    ck(cudaEventRecord(e_end, s_gpu_), "record");
    ck(cudaEventSynchronize(e_end), "sync");
    if (coll_) coll_->check();  // an asynchronous collective failure surfaces here
    const double host_end = std::chrono::duration<double>(std::chrono::steady_clock::now() - host_t0).count();
    std::memcpy(out, h_tok_ + static_cast<size_t>(max_steps_) * N_ * 3, static_cast<size_t>(steps) * N_ * 4);
    for (int i = 0; i < N_; ++i) pos_[i] += steps;
    capture_step_ = 0;  // the router tap covers one decode call

    // ---- measured timeline ----
    // Host (steady_clock) and GPU timers drift by tens of ppm; map host times
    // onto the device timebase with the two synchronisation points (e0 at
    // host 0, e_end at host_end).
    float total_ms = 0;
    ck(cudaEventElapsedTime(&total_ms, e0, e_end), "elapsed");
    const double clock_scale = host_end > 0 ? (total_ms * 1e-3) / host_end : 1.0;
    Timeline tl;
    tl.entries.resize(n);
    ScheduleDag measured = dag;
    for (int i = 0; i < n; ++i) {
        double s, e;
        if (ev_start[i]) {
            float a = 0, b = 0;
            ck(cudaEventElapsedTime(&a, e0, ev_start[i]), "elapsed");
            ck(cudaEventElapsedTime(&b, e0, ev_end[i]), "elapsed");
            s = a * 1e-3;
            e = b * 1e-3;
        } else {
            s = h_start[i] * clock_scale;
            e = h_end[i] * clock_scale;
        }
        tl.entries[i] = {i, s, e};
        measured.tasks[i].duration = e - s;
        tl.busy[static_cast<int>(measured.tasks[i].resource)] += e - s;
        tl.makespan = std::max(tl.makespan, e);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e_end);
    cudaEventDestroy(e_inputs);

    DecodeReport rep;  // (the per-kernel event breakdown is read on demand: kernel_events())
    {  // in-kernel execution times of the GEMMs
        std::vector<unsigned long long> tv(2 * ktime_names_.size());
        if (!tv.empty())
            ck(cudaMemcpy(tv.data(), d_ktime_, tv.size() * 8, cudaMemcpyDeviceToHost), "timers");
        for (size_t k = 0; k < ktime_names_.size(); ++k) {
            const unsigned long long t0 = tv[2 * k], t1 = ~tv[2 * k + 1];
            if (t0 == ~0ull || t1 < t0) continue;  // launch had no work
            auto it = std::find_if(rep.kernel_exec.begin(), rep.kernel_exec.end(),
                                   [&](const DecodeReport::KernelTime& kt) { return kt.name == ktime_names_[k]; });
            if (it == rep.kernel_exec.end()) {
                rep.kernel_exec.push_back({ktime_names_[k], 0.0, 0});
                it = rep.kernel_exec.end() - 1;
            }
            it->ms += (t1 - t0) * 1e-6;
            it->launches += 1;
        }
    }
    for (const auto& kt : rep.kernel_exec) {
        if (kt.name == "expert_gateup_gemm" || kt.name == "expert_down_gemm") rep.expert_ms_total += kt.ms;
        if (kt.name == "expert_gateup_gemm") rep.expert_launches = kt.launches;
        if (kt.name == "qkv_gemm" || kt.name == "o_gemm") {
            rep.qkv_o_ms_total += kt.ms;
            rep.dense_launches += kt.launches;
        }
    }
    rep.seconds = total_ms * 1e-3;
    rep.tokens_per_second = static_cast<double>(N_) * steps / rep.seconds;
    rep.gpu_launches = launches_;
    const double layers = static_cast<double>(L_) * steps;
    for (int i = 0; i < n; ++i) {
        const Task& t = measured.tasks[i];
        switch (t.kind) {
            case TaskKind::PreAttn:
            case TaskKind::GpuAttn: rep.measured.gpu_attention += t.duration / layers; break;
            case TaskKind::PostAttn: rep.measured.gpu_ffn += t.duration / layers; break;
            case TaskKind::CpuAttn: rep.measured.cpu_attention += t.duration / layers; break;
            case TaskKind::WeightToGpu: {
                rep.measured.link_upload += t.duration / layers;
                const auto [b, e] = page_range(t.page);
                rep.h2d_weight_bytes += static_cast<double>(e - b);
                rep.h2d_bytes += static_cast<double>(e - b);
                break;
            }
            case TaskKind::LoadHidden:
                rep.measured.link_upload += t.duration / layers;
                rep.h2d_bytes += static_cast<double>(Rmu_) * Ho_ * 2;  // this rank's heads (act_load_hidden)
                break;
            case TaskKind::OffloadQkv: rep.d2h_bytes += static_cast<double>(mu_) * W_ * 2; break;
            default: break;
        }
    }
    // Host/device clock alignment error is bounded by the e0 synchronisation
    // latency; verify with 50 us slack.
    rep.verify = lightplan::sim::verify_timeline_tol(measured, tl, 5e-5);
    const auto m = lightplan::sim::metrics(measured, tl);
    rep.steady_layer_time = m.steady_layer_time;
    rep.measured.layer_total = m.steady_layer_time;
    for (int r = 0; r < 5; ++r) rep.utilization[r] = m.utilization[r];
    if (dag_out) *dag_out = std::move(measured);
    if (tl_out) *tl_out = std::move(tl);
    if (const char* ht = std::getenv("MLT_HOST_TIMING"); ht && ht[0] == '1') {
        const double tot = std::chrono::duration<double>(std::chrono::steady_clock::now() - call_t0).count();
        std::fprintf(stderr, "[mlt] decode call host phases: setup %.1f ms, device region %.1f ms, report %.1f ms\n",
                     setup_s * 1e3, host_end * 1e3, (tot - setup_s - host_end) * 1e3);
    }
    return rep;
}

}  // namespace mlt
