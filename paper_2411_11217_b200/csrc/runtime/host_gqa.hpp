// Host-core GQA decode attention (A_g = 0): the
// CpuAttn task of the CGOPipe DAG (pipesim.hpp:26).  KV layout per (seq, kv
// head): kD-wide bf16 rows, one contiguous stream of max_ctx rows for K and
// one for V (host_attention.cpp).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace mlt {

// One (sequence, kv head): the G query heads q[G][128] (bf16) against the L
// rows of kc / vc; out[G][128] bf16.  sc: host_gqa_scratch_floats(max_ctx)
// floats of scratch, ldsc = host_gqa_ldsc(max_ctx), L <= max_ctx.
void host_gqa_item(const uint16_t* q, const uint16_t* kc, const uint16_t* vc, int L, int G, float scale,
                   float* sc, int ldsc, uint16_t* out);

// T sequences: q [T][nq][128] bf16, kc / vc [T][nkv][max_ctx][128] bf16,
// ctx[t] valid rows, out [T][nq][128] bf16; threads <= 0 = all host cores.
void host_gqa_decode(const uint16_t* q, const uint16_t* kc, const uint16_t* vc, const int32_t* ctx, int T,
                     int nq, int nkv, int max_ctx, uint16_t* out, int threads);

bool host_gqa_bf16dot();
int host_gqa_ldsc(int max_ctx);
size_t host_gqa_scratch_floats(int max_ctx);
// AMX tile path (scores and P.V on the tile unit) when the CPU has AMX-BF16
// and the kernel grants the tile state; MLT_HOST_AMX=0 or set_amx(false)
// selects the AVX-512 path.  set_amx returns whether AMX is now in use.
bool host_gqa_amx();
bool host_gqa_set_amx(bool enable);

// Host core plan for one decode: the first two cores of the process's
// affinity mask run the resource launcher threads (GPU, H2D, D2H, pinning
// workers of the executor), the rest run the attention team, split evenly
// between the `sharing` co-located TP ranks (`rank`'s slice).  With fewer
// than four cores nothing is pinned (attn = all cores, launch empty).
struct HostCores {
    std::vector<int> launch, attn;
    bool pinned = false;
};
HostCores host_cores(int rank, int sharing);
// Restrict the calling thread to `cores` (no-op for an empty set).
void pin_thread(const std::vector<int>& cores);

}  // namespace mlt
