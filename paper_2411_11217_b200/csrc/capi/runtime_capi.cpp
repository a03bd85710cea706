// C ABI over mlt::Runtime (include/mlt.h, "Decode runtime").
#include <memory>
#include <string>

#include <cstring>
#include <vector>

#include "../kernels/common.cuh"
#include "../runtime/host_layout.hpp"
#include "../runtime/runtime.hpp"
#include "lightplan/pipesim.hpp"
#include "lightplan/planner.hpp"
#include "lightplan/batcher.hpp"
#include "status.hpp"

namespace {

template <class F>
int guard(F&& f) {
    MLT_GUARD_BODY(lightplan)
}

struct Handle {
    std::unique_ptr<mlt::Runtime> rt;
    lightplan::sim::ScheduleDag dag;
    lightplan::sim::Timeline tl;
    bool has_tl = false;
    std::vector<mlt::DecodeReport::KernelTime> kernels, kernel_exec;
    bool kernels_fresh = true;  // kernels holds the last decode call's event breakdown
};

Handle* H(mlt_runtime* r) { return reinterpret_cast<Handle*>(r); }

}  // namespace

extern "C" {

mlt_runtime* mlt_runtime_create_with_weights(const mlt_model_spec_t* m, const mlt_policy_t* p,
                                             const mlt_runtime_options_t* o, mlt_weight_fn get, void* ctx);

mlt_runtime* mlt_runtime_create(const mlt_model_spec_t* m, const mlt_policy_t* p,
                                const mlt_runtime_options_t* o) {
    return mlt_runtime_create_with_weights(m, p, o, nullptr, nullptr);
}

mlt_runtime* mlt_runtime_create_with_weights(const mlt_model_spec_t* m, const mlt_policy_t* p,
                                             const mlt_runtime_options_t* o, mlt_weight_fn get, void* ctx) {
    Handle* h = nullptr;
    guard([&] {
        lightplan::ModelSpec ms;
        ms.layers = m->layers; ms.hidden_dim = m->hidden_dim; ms.ffn_dim = m->ffn_dim;
        ms.q_heads = m->q_heads; ms.kv_heads = m->kv_heads; ms.experts = m->experts;
        ms.top_k = m->top_k; ms.weight_dtype_bytes = m->weight_dtype_bytes;
        ms.kv_dtype_bytes = m->kv_dtype_bytes;
        lightplan::Policy pol;
        pol.batch = p->batch; pol.micro_batch = p->micro_batch;
        pol.attn_on_gpu = p->attn_on_gpu != 0; pol.ffn_on_gpu = p->ffn_on_gpu != 0;
        pol.weights_on_gpu = p->weights_on_gpu; pol.kv_on_gpu = p->kv_on_gpu;
        mlt::ModelExt ext;
        ext.vocab = o->vocab; ext.rms_eps = o->rms_eps; ext.rope_theta = o->rope_theta;
        ext.lm_head_scale = o->lm_head_scale; ext.seed = o->seed;
        mlt::RuntimeOptions opt;
        opt.device = o->device; opt.budget_bytes = o->budget_bytes; opt.max_ctx = o->max_ctx;
        opt.host_threads = o->host_threads; opt.pin_weights = o->pin_weights;
        opt.exact_gates = o->exact_gates;
        opt.tp_rank = o->tp_size > 1 ? o->tp_rank : 0;
        opt.tp_size = o->tp_size > 1 ? o->tp_size : 1;
        std::memcpy(opt.nccl_id, o->nccl_id, 128);
        opt.schedule = o->schedule;
        opt.prefill_chunk_tokens = o->prefill_chunk_tokens;
        opt.tp_shard_only = o->tp_shard_only != 0;
        opt.weight_codec = o->weight_codec != 0;
        opt.pdl = o->disable_pdl == 0;
        opt.expert_down_splits = o->expert_down_splits;
        opt.collective = o->collective;
        opt.weight_fn = get;
        opt.weight_ctx = ctx;
        auto hh = std::make_unique<Handle>();
        hh->rt = std::make_unique<mlt::Runtime>(ms, ext, pol, opt);
        h = hh.release();
        return MLT_OK;
    });
    return reinterpret_cast<mlt_runtime*>(h);
}

void mlt_runtime_destroy(mlt_runtime* r) { delete H(r); }

namespace {
lightplan::ModelSpec model_in(const mlt_model_spec_t* m) {
    lightplan::ModelSpec ms;
    ms.layers = m->layers; ms.hidden_dim = m->hidden_dim; ms.ffn_dim = m->ffn_dim;
    ms.q_heads = m->q_heads; ms.kv_heads = m->kv_heads; ms.experts = m->experts;
    ms.top_k = m->top_k; ms.weight_dtype_bytes = m->weight_dtype_bytes;
    ms.kv_dtype_bytes = m->kv_dtype_bytes;
    return ms;
}
}  // namespace

int mlt_tp_shard(const mlt_model_spec_t* m, int rank, int size, mlt_tp_shard_t* out) {
    return guard([&] {
        const mlt::Shard s = mlt::make_shard(model_in(m), rank, size);
        *out = {s.q_heads, s.kv_heads, s.ffn, s.qkv_rows, s.o_k, s.ffn_off};
        return MLT_OK;
    });
}

int mlt_synth_tp_weight(const mlt_model_spec_t* m, int rank, int size, uint64_t seed, int layer,
                        int kind, int expert, uint16_t* out, int64_t* rows, int64_t* cols) {
    return guard([&] {
        const lightplan::ModelSpec ms = model_in(m);
        const mlt::Shard s = mlt::make_shard(ms, rank, size);
        const mlt::ShardMap sm = mlt::shard_map(ms, s, kind);
        const int64_t R = static_cast<int64_t>(sm.rows.size());
        *rows = R;
        *cols = sm.k_local;
        if (!out) return MLT_OK;
        std::vector<uint16_t> packed(static_cast<size_t>(R) * sm.k_local);
        mlt::synth_shard_packed(seed, mlt::tensor_id(layer, kind, expert), sm.k_global, sm.rows.data(), sm.col0,
                                sm.k_local, 0, R, sm.scale, packed.data());
        // unpack [R, K] (block-major A layout) for inspection
        const uint8_t* p = reinterpret_cast<const uint8_t*>(packed.data());
        for (int64_t i = 0; i < R; ++i)
            for (int64_t k = 0; k < sm.k_local; ++k)
                std::memcpy(out + i * sm.k_local + k, p + mltk::a_packed_off(i, k, sm.k_local), 2);
        return MLT_OK;
    });
}

int mlt_nccl_unique_id(uint8_t out[128]) {
    return guard([&] {
        mlt::nccl_unique_id(out);
        return MLT_OK;
    });
}

mlt_dag* mlt_execution_dag(const mlt_dag* ref, const mlt_model_spec_t* m, const mlt_policy_t* p,
                           int exact_gates, mlt_runtime_info_t* info) {
    mlt_dag* out = nullptr;
    guard([&] {
        lightplan::ModelSpec ms;
        ms.layers = m->layers; ms.hidden_dim = m->hidden_dim; ms.ffn_dim = m->ffn_dim;
        ms.q_heads = m->q_heads; ms.kv_heads = m->kv_heads; ms.experts = m->experts;
        ms.top_k = m->top_k; ms.weight_dtype_bytes = m->weight_dtype_bytes;
        ms.kv_dtype_bytes = m->kv_dtype_bytes;
        lightplan::Policy pol;
        pol.batch = p->batch; pol.micro_batch = p->micro_batch;
        pol.attn_on_gpu = p->attn_on_gpu != 0; pol.ffn_on_gpu = p->ffn_on_gpu != 0;
        pol.weights_on_gpu = p->weights_on_gpu; pol.kv_on_gpu = p->kv_on_gpu;
        const auto& dag = *reinterpret_cast<const lightplan::sim::ScheduleDag*>(ref);
        const mlt::Catalog cat = mlt::build_catalog(ms, pol);
        auto* d = new lightplan::sim::ScheduleDag(
            mlt::execution_dag(dag, cat, static_cast<int>(pol.micro_batch_count()), exact_gates != 0));
        if (info) {
            info->achieved_weight_ratio = cat.achieved_rw;
            info->streamed_bytes_per_layer = static_cast<double>(cat.blob_bytes);
            info->arena_used = info->arena_capacity = info->pin_seconds = info->gen_seconds = 0;
            info->bytes_per_weight = info->raw_blocks = info->codec_engine = 0;
        }
        out = reinterpret_cast<mlt_dag*>(d);
        return MLT_OK;
    });
    return out;
}

int mlt_runtime_info(const mlt_runtime* r, mlt_runtime_info_t* out) {
    return guard([&] {
        const auto& rt = *reinterpret_cast<const Handle*>(r)->rt;
        out->achieved_weight_ratio = rt.achieved_weight_ratio();
        out->streamed_bytes_per_layer = static_cast<double>(rt.streamed_bytes_per_layer());
        out->arena_used = static_cast<double>(rt.arena_used());
        out->arena_capacity = 0;
        out->pin_seconds = rt.pin_seconds();
        out->gen_seconds = rt.gen_seconds();
        out->bytes_per_weight = rt.bytes_per_weight();
        out->raw_blocks = static_cast<double>(rt.raw_blocks());
        out->codec_engine = static_cast<double>(rt.codec_mode());
        return MLT_OK;
    });
}

int mlt_runtime_prefill_synthetic(mlt_runtime* r, int prompt_len, uint64_t seed) {
    return guard([&] {
        H(r)->rt->prefill_synthetic(prompt_len, seed);
        return MLT_OK;
    });
}

int mlt_runtime_prefill(mlt_runtime* r, const int32_t* tokens, const int32_t* lens, int32_t* first_ids,
                        mlt_prefill_report_t* rep) {
    return guard([&] {
        const mlt::PrefillReport p = H(r)->rt->prefill(tokens, lens, first_ids);
        if (rep)
            *rep = {p.seconds, p.tokens_per_second, p.prompt_tokens, p.chunk_tokens, p.chunks_per_layer,
                    p.h2d_weight_bytes, p.h2d_bytes, p.d2h_bytes, p.gpu_busy_seconds, p.gpu_launches};
        return MLT_OK;
    });
}

int mlt_runtime_set_positions(mlt_runtime* r, const int32_t* pos) {
    return guard([&] {
        H(r)->rt->set_positions(pos);
        return MLT_OK;
    });
}

int mlt_runtime_decode(mlt_runtime* r, const int32_t* tokens, const int32_t* forced, int steps,
                       int32_t* out, mlt_decode_report_t* rep) {
    return guard([&] {
        Handle* h = H(r);
        const mlt::DecodeReport d = h->rt->decode(tokens, forced, steps, out, &h->dag, &h->tl);
        h->has_tl = true;
        h->kernels_fresh = false;
        h->kernel_exec = d.kernel_exec;
        if (rep) {
            rep->seconds = d.seconds;
            rep->tokens_per_second = d.tokens_per_second;
            rep->measured = {d.measured.link_upload, d.measured.gpu_attention, d.measured.gpu_ffn,
                             d.measured.cpu_attention, d.measured.cpu_ffn, d.measured.layer_total};
            rep->h2d_weight_bytes = d.h2d_weight_bytes;
            rep->h2d_bytes = d.h2d_bytes;
            rep->d2h_bytes = d.d2h_bytes;
            rep->steady_layer_time = d.steady_layer_time;
            for (int i = 0; i < 5; ++i) rep->utilization[i] = d.utilization[i];
            rep->gpu_launches = d.gpu_launches;
            rep->timeline_ok = d.verify.empty() ? 1 : 0;
            rep->expert_ms_total = d.expert_ms_total;
            rep->expert_launches = d.expert_launches;
            rep->dense_ms_total = d.qkv_o_ms_total;
            rep->dense_launches = d.dense_launches;
        }
        if (!d.verify.empty()) mlt::set_error(("timeline: " + d.verify).c_str(), MLT_OK);
        return MLT_OK;
    });
}

int mlt_runtime_execute(mlt_runtime* r, const mlt_dag* dag, const int32_t* tokens, const int32_t* forced,
                        int32_t* out, mlt_decode_report_t* rep) {
    return guard([&] {
        if (!dag) throw std::invalid_argument("execute: null dag");
        Handle* h = H(r);
        const auto& d0 = *reinterpret_cast<const lightplan::sim::ScheduleDag*>(dag);
        const mlt::DecodeReport d = h->rt->execute(d0, tokens, forced, out, &h->dag, &h->tl);
        h->has_tl = true;
        h->kernels_fresh = false;
        h->kernel_exec = d.kernel_exec;
        if (rep) {
            rep->seconds = d.seconds;
            rep->tokens_per_second = d.tokens_per_second;
            rep->measured = {d.measured.link_upload, d.measured.gpu_attention, d.measured.gpu_ffn,
                             d.measured.cpu_attention, d.measured.cpu_ffn, d.measured.layer_total};
            rep->h2d_weight_bytes = d.h2d_weight_bytes;
            rep->h2d_bytes = d.h2d_bytes;
            rep->d2h_bytes = d.d2h_bytes;
            rep->steady_layer_time = d.steady_layer_time;
            for (int i = 0; i < 5; ++i) rep->utilization[i] = d.utilization[i];
            rep->gpu_launches = d.gpu_launches;
            rep->timeline_ok = d.verify.empty() ? 1 : 0;
            rep->expert_ms_total = d.expert_ms_total;
            rep->expert_launches = d.expert_launches;
            rep->dense_ms_total = d.qkv_o_ms_total;
            rep->dense_launches = d.dense_launches;
        }
        return MLT_OK;
    });
}

int mlt_runtime_kernel_profile(mlt_runtime* r, char* buf, size_t cap) {
    return guard([&] {
        std::string s = "{";
        char line[256];
        const char* keys[2] = {"events", "exec"};
        if (!H(r)->kernels_fresh) {  // event deltas read on demand (Runtime::kernel_events)
            H(r)->kernels = H(r)->rt->kernel_events();
            H(r)->kernels_fresh = true;
        }
        const std::vector<mlt::DecodeReport::KernelTime>* lists[2] = {&H(r)->kernels, &H(r)->kernel_exec};
        for (int L = 0; L < 2; ++L) {
            s += std::string(L ? "," : "") + "\"" + keys[L] + "\":[";
            for (size_t i = 0; i < lists[L]->size(); ++i) {
                const auto& k = (*lists[L])[i];
                std::snprintf(line, sizeof line, "%s{\"name\":\"%s\",\"ms\":%.6f,\"launches\":%d}", i ? "," : "",
                              k.name.c_str(), k.ms, k.launches);
                s += line;
            }
            s += "]";
        }
        s += "}";
        if (buf && cap) {
            const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
        return static_cast<int>(s.size());
    });
}

int mlt_runtime_timeline_json(mlt_runtime* r, char* buf, size_t cap) {
    return guard([&] {
        Handle* h = H(r);
        if (!h->has_tl) throw std::invalid_argument("no decode has run yet");
        const std::string s = lightplan::sim::timeline_json(h->dag, h->tl, "{\"source\":\"measured\"}");
        if (buf && cap) {
            const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
        return static_cast<int>(s.size());
    });
}

int mlt_runtime_read_residual(mlt_runtime* r, float* out) {
    return guard([&] {
        H(r)->rt->read_residual(out);
        return MLT_OK;
    });
}

int mlt_runtime_capture_router(mlt_runtime* r, int step) {
    return guard([&] {
        H(r)->rt->capture_router(step);
        return MLT_OK;
    });
}

int mlt_runtime_debug_read(mlt_runtime* r, const char* name, void* out, size_t cap) {
    return guard([&] { return static_cast<int>(H(r)->rt->debug_read(name, out, cap)); });
}

}  // extern "C"
