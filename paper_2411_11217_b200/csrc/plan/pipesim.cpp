// CGOPipe / S2 / S3 / S4 schedule construction, list-scheduling simulator,
// metrics and invariant checker.
//
// Schedules are expressed over global micro-batch slots q = (g-1)*M + j
// (g = global layer across all decode steps, j = micro-batch within the
// layer), exactly the indexing of proj/src/pipesim.cpp:59-63.  The issue
// recipes restate pipesim.cpp:196-273; the resulting
// task list is compared edge-for-edge with the compiled reference in
// tests/test_schedule_parity.py.  The B200 executor (runtime/executor.cpp)
// consumes this list unchanged: per-resource FIFO in issue order.
#include "lightplan/pipesim.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>

#include "lightplan/opcost.hpp"

namespace lightplan::sim {

const char* to_string(TaskKind k) {
    static const char* const n[] = {"pre_attn",    "offload_qkv",      "cpu_attn",
                                    "load_hidden", "post_attn",        "weight_to_pinned",
                                    "weight_to_gpu", "kv_load",        "gpu_attn"};
    const int i = static_cast<int>(k);
    return (i >= 0 && i < 9) ? n[i] : "unknown";
}

const char* to_string(Resource r) {
    static const char* const n[] = {"gpu", "cpu", "h2d", "d2h", "ctopin"};
    const int i = static_cast<int>(r);
    return (i >= 0 && i < kResourceCount) ? n[i] : "unknown";
}

ScheduleKind parse_schedule_kind(const std::string& s) {
    if (s == "cgopipe") return ScheduleKind::CgoPipe;
    if (s == "s2") return ScheduleKind::S2;
    if (s == "s3") return ScheduleKind::S3;
    if (s == "s4") return ScheduleKind::S4;
    throw std::invalid_argument("unknown schedule kind: " + s);
}

const char* to_string(ScheduleKind k) {
    switch (k) {
        case ScheduleKind::CgoPipe: return "cgopipe";
        case ScheduleKind::S2: return "s2";
        case ScheduleKind::S3: return "s3";
        case ScheduleKind::S4: return "s4";
    }
    return "unknown";
}

namespace {

constexpr int kNone = -1;

// Task-id tables indexed by slot (1-based) or by global layer.
struct SlotTables {
    std::vector<int> pre, off, cpu, loadh, post, kv, gattn, page_up, page_pin;
    std::vector<int> layer_up, layer_pin;
    void size(long slots, int layers) {
        for (auto* v : {&pre, &off, &cpu, &loadh, &post, &kv, &gattn, &page_up, &page_pin})
            v->assign(slots + 1, kNone);
        layer_up.assign(layers + 1, kNone);
        layer_pin.assign(layers + 1, kNone);
    }
};

class Recipe {
  public:
    Recipe(const DurationProvider& dur, ScheduleKind kind, int layers, int steps, int m)
        : L_(layers), M_(m) {
        if (layers < 1 || steps < 1 || m < 1)
            throw std::invalid_argument("layers, steps and micro-batch count must be >= 1");
        G_ = layers * steps;
        S_ = static_cast<long>(G_) * m;
        per_step_.reserve(steps);
        for (int s = 1; s <= steps; ++s) per_step_.push_back(dur(s));
        out_.kind = kind;
        out_.layers = layers;
        out_.steps = steps;
        out_.micro_batches = m;
        t_.size(S_, G_);
    }

    ScheduleDag run() {
        switch (out_.kind) {
            case ScheduleKind::CgoPipe: cgopipe(); break;
            case ScheduleKind::S2: s2(); break;
            case ScheduleKind::S3: s3(); break;
            case ScheduleKind::S4: s4(); break;
        }
        gate_on_weights();
        return std::move(out_);
    }

  private:
    // --- slot arithmetic --------------------------------------------------
    int g_of(long q) const { return static_cast<int>((q - 1) / M_) + 1; }
    int j_of(long q) const { return static_cast<int>((q - 1) % M_) + 1; }
    bool slot_ok(long q) const { return q >= 1 && q <= S_; }
    bool layer_ok(int g) const { return g >= 1 && g <= G_; }
    const StepDurations& du(int g) const { return per_step_[(g - 1) / L_]; }

    int push(TaskKind k, Resource r, int g, int mb, int page, double dur, std::vector<int> deps) {
        Task t;
        t.kind = k;
        t.resource = r;
        t.step = (g - 1) / L_ + 1;
        t.layer = (g - 1) % L_ + 1;
        t.microbatch = mb;
        t.page = page;
        t.duration = dur;
        t.deps = std::move(deps);
        out_.tasks.push_back(std::move(t));
        return static_cast<int>(out_.tasks.size()) - 1;
    }

    // --- weight transfer ----------------------------------------------------
    void page_pin(long p) {
        if (!slot_ok(p)) return;
        const int g = g_of(p);
        t_.page_pin[p] = push(TaskKind::WeightToPinned, Resource::CpuToPinned, g, 0, j_of(p),
                              du(g).weight_stage / M_, {});
    }
    void page_up(long p) {
        if (!slot_ok(p)) return;
        const int g = g_of(p);
        t_.page_up[p] = push(TaskKind::WeightToGpu, Resource::HostToDevice, g, 0, j_of(p),
                             du(g).weight_upload / M_, {t_.page_pin[p]});
    }
    void whole_pin(int g) {
        if (!layer_ok(g)) return;
        t_.layer_pin[g] = push(TaskKind::WeightToPinned, Resource::CpuToPinned, g, 0, 0,
                               du(g).weight_stage, {});
    }
    void whole_up(int g) {
        if (!layer_ok(g)) return;
        t_.layer_up[g] = push(TaskKind::WeightToGpu, Resource::HostToDevice, g, 0, 0,
                              du(g).weight_upload, {t_.layer_pin[g]});
    }
    void kv_load(long q) {
        if (!slot_ok(q)) return;
        const int g = g_of(q);
        t_.kv[q] = push(TaskKind::KvLoad, Resource::HostToDevice, g, j_of(q), 0, du(g).kv_load, {});
    }

    // --- compute chain ------------------------------------------------------
    // PreAttn -> OffloadQkv -> CpuAttn; PreAttn waits on the same micro-batch's
    // PostAttn of the previous global layer (residual stream).
    void front(long q) {
        if (!slot_ok(q)) return;
        const int g = g_of(q), j = j_of(q);
        std::vector<int> deps;
        if (q > M_ && t_.post[q - M_] != kNone) deps.push_back(t_.post[q - M_]);
        t_.pre[q] = push(TaskKind::PreAttn, Resource::Gpu, g, j, 0, du(g).pre_attn, std::move(deps));
        t_.off[q] = push(TaskKind::OffloadQkv, Resource::DeviceToHost, g, j, 0, du(g).offload_qkv,
                         {t_.pre[q]});
        t_.cpu[q] = push(TaskKind::CpuAttn, Resource::Cpu, g, j, 0, du(g).cpu_attn, {t_.off[q]});
    }
    void load_hidden(long q) {
        const int g = g_of(q);
        t_.loadh[q] = push(TaskKind::LoadHidden, Resource::HostToDevice, g, j_of(q), 0,
                           du(g).load_hidden, {t_.cpu[q]});
    }
    void back(long q) {
        const int g = g_of(q);
        t_.post[q] = push(TaskKind::PostAttn, Resource::Gpu, g, j_of(q), 0, du(g).post_attn,
                          {t_.loadh[q]});
    }

    // --- recipes ------------------------------------------------------------
    void cgopipe() {
        const long ahead = std::min<long>(2, M_);
        for (long p = 1; p <= std::min<long>(M_, S_); ++p) {  // first layer's pages up front
            page_pin(p);
            page_up(p);
        }
        for (long a = 1; a <= ahead; ++a) {
            front(a);
            page_pin(M_ + a);
        }
        for (long q = 1; q <= S_; ++q) {
            load_hidden(q);
            page_up(q + M_);
            back(q);
            front(q + ahead);
            page_pin(q + M_ + ahead);
        }
    }

    void s2() {
        const long ahead = std::min<long>(2, M_);
        whole_pin(1);
        whole_up(1);
        for (long a = 1; a <= ahead; ++a) front(a);
        whole_pin(2);
        for (long q = 1; q <= S_; ++q) {
            const bool last = j_of(q) == M_;
            load_hidden(q);
            back(q);
            if (last) whole_up(g_of(q) + 1);
            front(q + ahead);
            if (last) whole_pin(g_of(q) + 2);
        }
    }

    void s3() {
        whole_pin(1);
        whole_up(1);
        for (long q = 1; q <= S_; ++q) {
            front(q);
            load_hidden(q);
            back(q);
            if (j_of(q) == M_) {
                whole_pin(g_of(q) + 1);
                whole_up(g_of(q) + 1);
            }
        }
    }

    void s4() {
        whole_pin(1);
        whole_up(1);
        kv_load(1);
        for (long q = 1; q <= S_; ++q) {
            const int g = g_of(q), j = j_of(q);
            std::vector<int> deps;
            if (q > M_) deps.push_back(t_.post[q - M_]);
            t_.pre[q] = push(TaskKind::PreAttn, Resource::Gpu, g, j, 0, du(g).pre_attn, std::move(deps));
            kv_load(q + 1);
            t_.gattn[q] = push(TaskKind::GpuAttn, Resource::Gpu, g, j, 0, du(g).gpu_attn,
                               {t_.pre[q], t_.kv[q]});
            t_.post[q] = push(TaskKind::PostAttn, Resource::Gpu, g, j, 0, du(g).post_attn,
                              {t_.gattn[q]});
            if (j == M_) {
                whole_pin(g + 1);
                whole_up(g + 1);
            }
        }
    }

    // Every GPU compute task of layer g waits for all of layer g's weights
    // (routing may touch any expert).  Added last because lookahead tasks
    // reference transfers that are issued after them.
    void gate_on_weights() {
        for (Task& t : out_.tasks) {
            if (t.kind != TaskKind::PreAttn && t.kind != TaskKind::PostAttn &&
                t.kind != TaskKind::GpuAttn)
                continue;
            const int g = (t.step - 1) * L_ + t.layer;
            if (t_.layer_up[g] != kNone) {
                t.deps.push_back(t_.layer_up[g]);
                continue;
            }
            for (long p = static_cast<long>(g - 1) * M_ + 1; p <= static_cast<long>(g) * M_; ++p)
                if (t_.page_up[p] != kNone) t.deps.push_back(t_.page_up[p]);
        }
    }

    int L_, M_, G_ = 0;
    long S_ = 0;
    std::vector<StepDurations> per_step_;
    ScheduleDag out_;
    SlotTables t_;
};

std::string g9(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.9g", v);
    return b;
}

}  // namespace

ScheduleDag build_schedule(const DurationProvider& durations, ScheduleKind kind, int layers,
                           int steps, int micro_batches) {
    return Recipe(durations, kind, layers, steps, micro_batches).run();
}

ScheduleDag build_schedule(const HardwareSpec& hw, const ModelSpec& model,
                           const WorkloadSpec& workload, const Policy& policy, ScheduleKind kind,
                           int layers, int steps) {
    // Placement rules of pipesim.cpp:302-314.
    if (kind == ScheduleKind::S4 && !policy.attn_on_gpu)
        throw UnsupportedCombinationError("s4 schedules GPU attention and requires A_g = 1");
    if (kind != ScheduleKind::S4 && policy.attn_on_gpu)
        throw UnsupportedCombinationError(std::string(to_string(kind)) +
                                          " schedules CPU attention and requires A_g = 0"
                                          " (with A_g = 1, use s4)");
    if (!policy.ffn_on_gpu)
        throw UnsupportedCombinationError(
            "pipeline schedules place the MoE FFN on the GPU and require F_g = 1");

    const int n_ub = static_cast<int>(policy.micro_batch_count());
    const double N = static_cast<double>(policy.batch);
    // Analytic durations: per-layer roofline terms split evenly over the
    // micro-batches (pipesim.cpp:319-346).
    auto model_durations = [=](int step) {
        const double ctx = static_cast<double>(workload.prompt_len + step);
        const OpProfile attn = attention_decode_profile(model, N, ctx);
        const OpProfile ffn = moe_ffn_profile(model, N, policy.weights_on_gpu);
        const ProjectionProfiles proj = projection_profiles(model, N);
        const TransferSizes xfer = transfer_sizes(model, policy, ctx);
        auto rt = [](double bytes, double bw, double flops, double peak) {
            return std::max(bytes / bw, flops / peak);
        };
        StepDurations s;
        s.pre_attn = rt(proj.qkv.gpu_bytes, hw.gpu_bw, proj.qkv.flops, hw.gpu_flops) / n_ub;
        s.post_attn = (rt(proj.output.gpu_bytes, hw.gpu_bw, proj.output.flops, hw.gpu_flops) +
                       rt(ffn.gpu_bytes, hw.gpu_bw, ffn.flops, hw.gpu_flops)) /
                      n_ub;
        if (policy.attn_on_gpu)
            s.gpu_attn = rt(attn.gpu_bytes, hw.gpu_bw, attn.flops, hw.gpu_flops) / n_ub;
        else
            s.cpu_attn = rt(attn.cpu_bytes, hw.cpu_bw, attn.flops, hw.cpu_flops) / n_ub;
        s.offload_qkv = xfer.qkv_offload / hw.link_bw;
        s.load_hidden = xfer.hidden_upload / hw.link_bw;
        s.weight_upload = xfer.weight_stream / hw.link_bw;
        s.weight_stage = xfer.weight_stream / hw.cpu_bw;
        s.kv_load = xfer.kv_upload / hw.link_bw;
        return s;
    };
    return build_schedule(model_durations, kind, layers, steps, n_ub);
}

Timeline simulate(const ScheduleDag& dag) {
    // Longest-path list scheduling over deps + per-resource FIFO chains,
    // evaluated by repeatedly draining each resource's queue head while its
    // dependencies are finished.  Start times equal the reference Kahn pass
    // (pipesim.cpp:350-406): both compute start = max(end of predecessors).
    const int n = static_cast<int>(dag.tasks.size());
    Timeline tl;
    tl.entries.resize(n);
    std::array<std::vector<int>, kResourceCount> fifo;
    for (int i = 0; i < n; ++i) {
        for (int dep : dag.tasks[i].deps)
            if (dep < 0 || dep >= n) throw CycleDetectedError("dependency index out of range");
        fifo[static_cast<int>(dag.tasks[i].resource)].push_back(i);
    }
    std::vector<char> done(n, 0);
    std::array<std::size_t, kResourceCount> head{};
    std::array<double, kResourceCount> free_at{};
    int finished = 0;
    for (bool moved = true; moved && finished < n;) {
        moved = false;
        for (int r = 0; r < kResourceCount; ++r) {
            while (head[r] < fifo[r].size()) {
                const int i = fifo[r][head[r]];
                const Task& t = dag.tasks[i];
                double ready = free_at[r];
                bool ok = true;
                for (int dep : t.deps) {
                    if (!done[dep]) { ok = false; break; }
                    ready = std::max(ready, tl.entries[dep].end);
                }
                if (!ok) break;
                tl.entries[i] = {i, ready, ready + t.duration};
                free_at[r] = ready + t.duration;
                tl.busy[r] += t.duration;
                tl.makespan = std::max(tl.makespan, ready + t.duration);
                done[i] = 1;
                ++finished;
                ++head[r];
                moved = true;
            }
        }
    }
    if (finished != n)
        throw CycleDetectedError("task graph has a cycle through deps or resource order");
    return tl;
}

SimMetrics metrics(const ScheduleDag& dag, const Timeline& tl) {
    if (dag.tasks.empty() || tl.entries.empty()) throw EmptyTimelineError("timeline has no tasks");
    SimMetrics m;
    m.makespan = tl.makespan;
    for (int r = 0; r < kResourceCount; ++r)
        m.utilization[r] = m.makespan > 0 ? tl.busy[r] / m.makespan : 0.0;

    const int G = dag.layers * dag.steps;
    std::vector<double> done_at(G + 1, 0.0);
    for (std::size_t i = 0; i < dag.tasks.size(); ++i) {
        const int g = (dag.tasks[i].step - 1) * dag.layers + dag.tasks[i].layer;
        done_at[g] = std::max(done_at[g], tl.entries[i].end);
    }
    // Interior layers only: 1-2 carry the fill, G the drain (pipesim.cpp:427-440).
    std::vector<double> gap;
    for (int g = 3; g + 1 <= G; ++g) gap.push_back(done_at[g] - done_at[g - 1]);
    if (gap.empty()) {
        m.steady_layer_time = m.makespan / G;
    } else {
        std::sort(gap.begin(), gap.end());
        const std::size_t h = gap.size() / 2;
        m.steady_layer_time = (gap.size() & 1) ? gap[h] : 0.5 * (gap[h - 1] + gap[h]);
    }
    return m;
}

std::string verify_timeline_tol(const ScheduleDag& dag, const Timeline& tl, double tol) {
    if (tl.entries.size() != dag.tasks.size()) return "entry count mismatch";
    std::ostringstream e;
    for (std::size_t i = 0; i < dag.tasks.size(); ++i) {
        const TimelineEntry& x = tl.entries[i];
        if (std::abs((x.end - x.start) - dag.tasks[i].duration) > tol) {
            e << "task " << i << ": span != duration";
            return e.str();
        }
        for (int dep : dag.tasks[i].deps)
            if (tl.entries[dep].end > x.start + tol) {
                e << "task " << i << ": starts before dependency " << dep << " ends";
                return e.str();
            }
    }
    std::array<std::vector<int>, kResourceCount> on;
    for (std::size_t i = 0; i < dag.tasks.size(); ++i)
        on[static_cast<int>(dag.tasks[i].resource)].push_back(static_cast<int>(i));
    for (auto& v : on) {
        std::sort(v.begin(), v.end(),
                  [&](int a, int b) { return tl.entries[a].start < tl.entries[b].start; });
        for (std::size_t k = 1; k < v.size(); ++k)
            if (tl.entries[v[k]].start + tol < tl.entries[v[k - 1]].end) {
                e << "tasks " << v[k - 1] << " and " << v[k] << " overlap on resource "
                  << to_string(dag.tasks[v[k]].resource);
                return e.str();
            }
    }
    return "";
}

std::string verify_timeline(const ScheduleDag& dag, const Timeline& tl) {
    return verify_timeline_tol(dag, tl, 1e-9);
}

std::string timeline_json(const ScheduleDag& dag, const Timeline& tl, const std::string& manifest) {
    const SimMetrics m = metrics(dag, tl);
    std::ostringstream o;
    o << "{\"manifest\":" << manifest << ",\"schedule\":\"" << to_string(dag.kind)
      << "\",\"tasks\":[";
    for (std::size_t i = 0; i < dag.tasks.size(); ++i) {
        const Task& t = dag.tasks[i];
        o << (i ? "," : "") << "{\"kind\":\"" << to_string(t.kind) << "\",\"step\":" << t.step
          << ",\"layer\":" << t.layer << ",\"microbatch\":" << t.microbatch
          << ",\"page\":" << t.page << ",\"resource\":\"" << to_string(t.resource)
          << "\",\"start\":" << g9(tl.entries[i].start) << ",\"end\":" << g9(tl.entries[i].end)
          << "}";
    }
    o << "],\"makespan\":" << g9(m.makespan) << ",\"utilization\":{";
    for (int r = 0; r < kResourceCount; ++r)
        o << (r ? "," : "") << "\"" << to_string(static_cast<Resource>(r))
          << "\":" << g9(m.utilization[r]);
    o << "},\"steady_layer_time\":" << g9(m.steady_layer_time) << "}";
    return o.str();
}

std::string timeline_csv(const ScheduleDag& dag, const Timeline& tl) {
    std::ostringstream o;
    o << "kind,step,layer,microbatch,page,resource,start,end\n";
    for (std::size_t i = 0; i < dag.tasks.size(); ++i) {
        const Task& t = dag.tasks[i];
        o << to_string(t.kind) << ',' << t.step << ',' << t.layer << ',' << t.microbatch << ','
          << t.page << ',' << to_string(t.resource) << ',' << g9(tl.entries[i].start) << ','
          << g9(tl.entries[i].end) << '\n';
    }
    return o.str();
}

}  // namespace lightplan::sim
