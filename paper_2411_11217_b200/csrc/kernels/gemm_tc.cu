// Weight-streaming grouped GEMM on tcgen05 / TMEM, fed by 1-D bulk copies
// from the paged weight pool.  One kernel serves every projection of the
// decode step:
//   * dense linears (QKV, O + residual, lm_head): G = 1, one matrix;
//   * expert gate/up (SURVEY.md §2c `expert_gateup_silu`): G = n_e experts,
//     two matrices (W1, W3) sharing the token operand, SiLU(g)*u fused in
//     the TMEM epilogue, written straight into the packed operand layout of
//     the down projection;
//   * expert down (`expert_down`): G = n_e, one matrix, fp32 rows per
//     (expert, token) slot for the deterministic top-k combine.
//
// Swap-AB: the weight rows fill UMMA M = 128, the (few) tokens of a group
// fill N in {16..256}; D^T = W X^T accumulates in TMEM (128 lanes x N fp32
// columns per matrix).  The kernel is HBM-bound at decode sizes (intensity
// mu*k/n_e << ridge), so the design goal is to keep every SM's copy queue
// full: warp 0 streams 16 KiB weight tiles (L2 evict_first) + the token tile
// (evict_last) into a multi-stage smem ring, warp 1 issues the MMAs from one
// elected lane and commits stages back, warps 2-5 drain TMEM.  Weight tiles
// are addressed through a page table (one pointer per row block), which is
// how the same kernel reads resident rows and rows paged into either pool
// slot (runtime/weights.cpp).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.hpp"

namespace mltk {
namespace {

constexpr int kThreadsRaw = 192;    // warp0 producer, warp1 MMA, warps2-5 epilogue
// Decoder group g (4 warps) owns the ring stages s with s % groups == g, so
// it meets each of its stages round after round and never waits on a stage
// barrier two phases ahead (mbarrier parity would alias).  Codec launches
// round the stage count to a multiple of the group count (GemmArgs::dec_groups,
// 2..kMaxDecGroups: more groups = more tiles decoding concurrently).
// 8 decoder warps (warps 6-13) form dec_groups groups: 2 groups of 128 threads
// alternate stages (each group decodes a whole stage), or 1 group of 256
// threads decodes every stage (half the per-stage decode latency).  3-4
// groups of 4 warps measured no faster (r02 profiles) and cost registers.
constexpr int kMaxDecGroups = 2;
constexpr int kDecWarpThreads = 256;
constexpr int kThreadsCodec = 192 + kDecWarpThreads;
// codec 3: + warp 14, the token-tile (B) producer
// codec 3: kTsGroups decoder groups of 4 warps (warps 6 .. 6 + 4 kTsGroups - 1)
// + the token-tile (B) producer warp after them
// codec 3 runs 3 decoder groups (4 measured no faster, 80 registers); the
// codec-4 decoder is more latency bound (dependent record loads) and gains
// from 4 groups: expert FFN at mu = 64 487 -> 462 us (profiles/r02s3_codec4.txt)
#ifndef MLT_TS_GROUPS_C4
#define MLT_TS_GROUPS_C4 4
#endif
__host__ __device__ constexpr int ts_groups(int codec) { return codec == 4 ? MLT_TS_GROUPS_C4 : 3; }
__host__ __device__ constexpr int ts_bwarp(int codec) { return 6 + 4 * ts_groups(codec); }
__host__ __device__ constexpr int ts_threads(int codec) { return 32 * (ts_bwarp(codec) + 1); }
constexpr int kCodecTile = 12432;   // encoded tile bytes (runtime/weight_codec.hpp)
constexpr int kCodec4Tile = 11600;  // codec 4 at the default capacity (GemmArgs::enc_tile)
__host__ __device__ inline int enc_tile_bytes(const GemmArgs& a) {
    return a.codec == 4 ? (a.enc_tile ? a.enc_tile : kCodec4Tile) : kCodecTile;
}
// codec: an encoded tile lands at the END of its 16 KiB A slot and is
// expanded in place (every input is in registers before any output store)
constexpr int kCodecOff = kATileBytes - kCodecTile;  // 3952, 16-byte aligned
constexpr int kMaxMats = 2;
constexpr int kEpiChunks = 1;           // 16-token TMEM chunks per load wait in the epilogue
constexpr int kCtlBytes = 1024;          // barriers + TMEM base
constexpr int kMaxRing = 16;             // codec 3: encoded-A ring slots / TMEM A slots
constexpr int kEpiScratch = 4 * 2048;    // per epilogue warp: 16 x 32 fp32 transpose tile

struct Smem {
    uint64_t full[kMaxRing];   // stage landed (codec 3: encoded A slot landed)
    uint64_t empty[kMaxRing];  // stage free (codec 3: encoded A slot read by its decoders)
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint64_t dfull[kMaxRing];  // codec 1: stage's A tiles decoded in place; codec 3: TMEM A slot written
    uint64_t aslot_empty[kMaxRing];  // codec 3: TMEM A slot consumed by the MMA
    uint64_t bfull[8], bempty[8];    // codec 3: token-tile ring
    uint32_t tmem_base;
};

static_assert(sizeof(Smem) <= kCtlBytes, "control block fits its reserved bytes");

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

// named barrier of one decoder group (ids 1.. ; 0 is __syncthreads)
template <int THR>
__device__ __forceinline__ void decoders_sync(int grp) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(THR) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Decode one encoded weight tile (weight_codec.hpp) into its 16 KiB bf16
// smem image; decoder thread dt handles the 8-weight units dt, dt +
// kDecThreads, ...  All of a thread's loads are issued first (ILP), then per
// 4 weights: two PRMT table lookups (codes 0-7 / 8-15 of the 16-byte
// table), a sign-replicating PRMT turning each code's bit 3 into a byte
// mask, one LOP3 select, and two PRMTs interleaving the raw low bytes with
// the looked-up high bytes: ~2.7 instructions per weight.
// PTX prmt.b32 (default mode): selector nibble bit 3 = replicate the sign of
// the selected byte (__byte_perm only documents the 3 low bits)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// high bytes of 4 weights: sel = their 3-bit table selectors (nibbles), m =
// 0xFF per byte where the code's bit 3 is set (from sign-replicating PRMT)
__device__ __forceinline__ uint32_t hi4(uint32_t sel, uint32_t m, const uint4& T) {
    const uint32_t a = prmt(T.x, T.y, sel);  // table[code & 7]
    const uint32_t b = prmt(T.z, T.w, sel);  // table[8 + (code & 7)]
    return (a & ~m) | (b & m);
}
// shared-window accesses by 32-bit smem address (generic pointers into
// dynamic smem compile to generic LD/ST, which cost extra latency and
// address math in the decoder's inner loop)
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const uint4& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// One decoder thread's share of an encoded tile: its units u = dt + j * THR
// (8 weights each), the table, and at most one escape entry.
template <int THR>
struct TileIn {
    uint4 T;
    uint2 lo[1024 / THR];
    uint32_t cd[1024 / THR];
    uint32_t n, esc;
};
template <int THR>
__device__ __forceinline__ void load_tile(uint32_t c, int dt, TileIn<THR>& in) {
    in.T = lds128(c + 12288);
    in.n = lds32(c + 12304) & 0xffffu;  // {u16 escape count, u16 0}
    in.esc = static_cast<uint32_t>(dt) < in.n ? lds32(c + 12308 + 4 * dt) : 0u;  // {u16 index, u8 hi, 0}
#pragma unroll
    for (int j = 0; j < 1024 / THR; ++j) {
        const uint32_t u = dt + j * THR;
        in.lo[j] = lds64(c + u * 8);
        in.cd[j] = lds32(c + 8192 + u * 4);
    }
}
template <int THR>
__device__ __forceinline__ void store_tile(const TileIn<THR>& in, uint32_t d, int dt) {
#pragma unroll
    for (int j = 0; j < 1024 / THR; ++j) {
        // code bit 3 of weight k sits at bit 4k+3: byte msbs of cd (odd k) and
        // of cd << 4 (even k) -> one sign-replicating PRMT per 4 weights
        const uint32_t cd = in.cd[j], c4 = cd << 4;
        const uint32_t h0 = hi4(cd & 0x7777u, prmt(c4, cd, 0xD9C8u), in.T);
        const uint32_t h1 = hi4((cd >> 16) & 0x7777u, prmt(c4, cd, 0xFBEAu), in.T);
        uint4 o;
        o.x = prmt(in.lo[j].x, h0, 0x5140u);
        o.y = prmt(in.lo[j].x, h0, 0x7362u);
        o.z = prmt(in.lo[j].y, h1, 0x5140u);
        o.w = prmt(in.lo[j].y, h1, 0x7362u);
        sts128(d + (dt + j * THR) * 16, o);
    }
}

// Page-table entries of an encoded (codec = 1) GEMM may carry tag bit 0: that
// 128-row block is stored as raw bf16 tiles (16 KiB each), the per-block
// fallback for weights the code cannot hold (runtime: codec_encode_tile
// fails) — copied straight into its A slot, never decoded.
__device__ __forceinline__ const uint8_t* untag(const uint8_t* p, bool& raw) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    raw = (u & 1u) != 0;
    return reinterpret_cast<const uint8_t*>(u & ~static_cast<uintptr_t>(1));
}

// Virtual task v -> (group, row block, token chunk, k-block range).  With
// the stream-K tail enabled, tasks past sk_full are (tail tile, K part).
struct VTask {
    int g, rb, c, kb0, kb1, part, tile;
};
__device__ __forceinline__ VTask vtask(const GemmArgs& a, int v, int KB) {
    VTask t;
    int u, ks, S;
    t.part = -1;
    t.tile = 0;
    if (a.sk_parts && v >= a.sk_full) {
        const int w = v - a.sk_full;
        t.tile = w / a.sk_parts;
        t.part = w % a.sk_parts;
        u = a.sk_full + t.tile;
        ks = t.part;
        S = a.sk_parts;
    } else {
        ks = v % a.k_splits;
        u = v / a.k_splits;
        S = a.k_splits;
    }
    t.c = u % a.n_chunks;
    t.g = (u / a.n_chunks) % a.G;
    t.rb = u / a.n_chunks / a.G;
    t.kb0 = ks * KB / S;
    t.kb1 = (ks + 1) * KB / S;
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// A stream-K part spins for its peers; the launch is cooperative (every CTA
// co-resident), so the wait always ends.  If it does not within this bound
// something is badly wrong: trap (a launch error) instead of hanging the GPU.
constexpr unsigned long long kSpinLimitNs = 2000000000ull;

// Decoder warps of a codec launch (warps 6-13): groups of THR threads own
// every (256 / THR)-th ring stage.  Per stage: every input (and escape entry)
// of the group's tiles -> registers, group barrier, expanded 16-byte stores
// over the same slots, escape bytes, proxy fence (generic smem writes ->
// tcgen05.mma), barrier, one arrive on the stage's dfull.
template <int THR>
__device__ __forceinline__ void decoder_role(const GemmArgs& a, uint8_t* smem, Smem* ctl, int stages, int stage_bytes,
                                             int kps, int n_virtual, int KB) {
    constexpr int kGroups = kDecWarpThreads / THR;
    const int grp = (static_cast<int>(threadIdx.x) - 192) / THR;
    const int dt = (static_cast<int>(threadIdx.x) - 192) % THR;
    int stage = 0, kstep = 0;
    uint32_t phase = 0;
    for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
        const VTask tk = vtask(a, v, KB);
        const int c = tk.c, g = tk.g, kb0 = tk.kb0, kb1 = tk.kb1;
        const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
        if (rows <= 0) continue;
        bool raw_m[kMaxMats] = {false, false};  // raw-fallback blocks: nothing to decode
        for (int mt = 0; mt < a.n_mats; ++mt)
            untag(a.a_table[(static_cast<int64_t>(mt) * a.G + tk.g) * a.RB + tk.rb], raw_m[mt]);
        for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
            for (int kb = kb0; kb < kb1; kb += kps, ++kstep) {
                // tiles of this stage: n_mats (one k-block) or kps (n_mats = 1), at most 2;
                // tile t belongs to matrix t (n_mats = 2) or matrix 0 (n_mats = 1)
                const bool two = a.n_mats * min(kps, kb1 - kb) == 2;
                const bool dec0 = !raw_m[0], dec1 = two && !raw_m[a.n_mats == 2 ? 1 : 0];
                if (stage % kGroups == grp) {
                    mbar_wait(&ctl->full[stage], phase);
                    if (a.ktrace && blockIdx.x == 0 && kstep < 256 && dt == 0) a.ktrace[256 + kstep] = globaltimer();
                    const uint32_t sa = smem_u32(smem + stage * stage_bytes);
                    TileIn<THR> in0, in1;
                    in0.n = in1.n = 0;
                    if (dec0) load_tile<THR>(sa + kCodecOff, dt, in0);
                    if (dec1) load_tile<THR>(sa + kATileBytes + kCodecOff, dt, in1);
                    decoders_sync<THR>(grp);  // all inputs read: the slots may be overwritten
                    if (dec0) store_tile<THR>(in0, sa, dt);
                    if (dec1) store_tile<THR>(in1, sa + kATileBytes, dt);
                    if (in0.n + in1.n) {  // rare: high bytes outside the table
                        decoders_sync<THR>(grp);
                        if (static_cast<uint32_t>(dt) < in0.n) sts8(sa + 2 * (in0.esc & 0xffffu) + 1, in0.esc >> 16);
                        if (static_cast<uint32_t>(dt) < in1.n)
                            sts8(sa + kATileBytes + 2 * (in1.esc & 0xffffu) + 1, in1.esc >> 16);
                    }
                    fence_proxy_async_smem();  // generic smem writes -> visible to tcgen05.mma
                    decoders_sync<THR>(grp);
                    if (a.ktrace && blockIdx.x == 0 && kstep < 256 && dt == 0) a.ktrace[512 + kstep] = globaltimer();
                    if (dt == 0) mbar_arrive(&ctl->dfull[stage]);
                }
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
        }
    }
}

// ---- codec 3: decode into tensor memory -----------------------------------
// Decoder thread (warp w, lane) owns row r = 32 (w % 4) + lane of a tile —
// the TMEM lane quarter warp w may access — and expands that row's 64
// weights (row-plane order, weight_codec.hpp rows_from_packed: 4 x 16-byte
// low-byte words + 4 x 8-byte code words, lane-consecutive) into the 32 TMEM
// columns of lane r (k pairs per 32-bit column, the A-operand layout of
// tcgen05.mma with A in TMEM).  No shared-memory writes: the A operand
// never returns to smem, the MMA reads it from TMEM.
__device__ __forceinline__ void decode_row_ts(uint32_t c, uint32_t r, uint32_t (&o)[32]) {
    const uint4 T = lds128(c + 12288);
    const uint32_t n = lds32(c + 12304) & 0xffffu;
    uint4 lo[4];
    uint2 cd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        lo[j] = lds128(c + (j * 128u + r) * 16u);
        cd[j] = lds64(c + 8192u + (j * 128u + r) * 8u);
    }
    // escapes (n <= 31): lane e holds entry e {u16 index, u8 high byte}
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t my_ent = lane < n ? lds32(c + 12308u + 4u * lane) : 0u;
    // branch-free expansion of the 8 units (independent: full ILP)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t cw = h ? cd[j].y : cd[j].x, c4 = cw << 4;
            const uint32_t h0 = hi4(cw & 0x7777u, prmt(c4, cw, 0xD9C8u), T);
            const uint32_t h1 = hi4((cw >> 16) & 0x7777u, prmt(c4, cw, 0xFBEAu), T);
            const uint32_t l0 = h ? lo[j].z : lo[j].x, l1 = h ? lo[j].w : lo[j].y;
            o[8 * j + 4 * h + 0] = prmt(l0, h0, 0x5140u);
            o[8 * j + 4 * h + 1] = prmt(l0, h0, 0x7362u);
            o[8 * j + 4 * h + 2] = prmt(l1, h1, 0x5140u);
            o[8 * j + 4 * h + 3] = prmt(l1, h1, 0x7362u);
        }
    }
    // patch escaped high bytes (rare; n is tile-uniform, so the loop is warp-uniform):
    // weight k of row r is the (k & 1) half of column k / 2
    for (uint32_t e = 0; e < n; ++e) {
        const uint32_t ent = __shfl_sync(0xffffffffu, my_ent, e), i = ent & 0xffffu;
        if (((i >> 4) & 127u) == r) {
            const uint32_t k = (i >> 11) * 16u + (i & 15u), col = k >> 1, sh = (k & 1u) * 16u + 8u;
            const uint32_t m = ~(0xffu << sh), hv = ((ent >> 16) & 0xffu) << sh;
#pragma unroll
            for (uint32_t q = 0; q < 32; ++q)
                if (q == col) o[q] = (o[q] & m) | hv;
        }
    }
}
// ---- codec 4: 3-bit codes (runtime/weight_codec.hpp codec4_encode_rows_tile) ----
// Same row ownership and TMEM layout as decode_row_ts.  Per 32 weights of a
// row: words A, B, C hold 24 codes in nibbles (bits 0-2; selector = word &
// 0x7777) and, in their nibble bit 3, the 3 bits of the last 8 codes,
// gathered into a fourth selector word by 3 shifts and 3 masked ORs.  One
// PRMT looks up 4 high bytes in this row's 8-byte table — slots 0-6 of the
// tile, slot 7 = the row's byte, or in the units its record flags the
// record's byte for that row half (one SEL per 4 weights) — two PRMTs interleave them with the
// raw low bytes, one subtraction per 2 weights undoes the tile's exponent
// phase: ~1.9 instructions per weight, all register indices static.  The
// rare hard escapes (~0.5 per row quarter) are patched by a warp-uniform
// loop with a predicated 32-way select.
struct EscC4 {
    uint32_t n, e0, e1;  // this warp's hard escapes: count, entries lane and 32 + lane
};

__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

template <bool kPhase>
__device__ __forceinline__ void expand_row_c4(const uint4 (&lo)[4], const uint32_t (&cw)[6], uint32_t t0, uint32_t t1,
                                              uint32_t t1x0, uint32_t t1x1, uint32_t rec, uint32_t (&o)[32]) {
#pragma unroll
    for (int H = 0; H < 2; ++H) {
        const uint32_t t1x = H ? t1x1 : t1x0;
        const uint32_t A = cw[3 * H], B = cw[3 * H + 1], C = cw[3 * H + 2];
        const uint32_t S = ((A >> 3) & 0x11111111u) | ((B >> 2) & 0x22222222u) | ((C >> 1) & 0x44444444u);
        const uint32_t sel[8] = {A & 0x7777u, (A >> 16) & 0x7777u, B & 0x7777u, (B >> 16) & 0x7777u,
                                 C & 0x7777u, (C >> 16) & 0x7777u, S, S >> 16};
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // weights k = 32H + 4u .. +3: unit 8H + u
#ifndef MLT_DIAG_C4_NOSEL
            const uint32_t tu = (rec >> (8 * H + u)) & 1u ? t1x : t1;
#else
            const uint32_t tu = t1 ^ (t1x & rec & 0);
#endif
            const uint32_t h4 = prmt(t0, tu, sel[u]);
            const uint4& l = lo[2 * H + (u >> 2)];
            const uint32_t lw = (u & 3) == 0 ? l.x : (u & 3) == 1 ? l.y : (u & 3) == 2 ? l.z : l.w;
            uint32_t x = prmt(lw, h4, 0x5140u), y = prmt(lw, h4, 0x7362u);
            if (kPhase) x -= 0x00800080u, y -= 0x00800080u;
            o[16 * H + 2 * u] = x;
            o[16 * H + 2 * u + 1] = y;
        }
    }
}

__device__ __forceinline__ void decode_row_c4(uint32_t c, uint32_t r, uint32_t (&o)[32], EscC4& esc) {
    // issue order matters (the loads are ordered volatile asm): the tile
    // header, this row's bytes, then the record / escape loads whose
    // addresses need the header, so their latency overlaps the row loads
    const uint2 T = lds64(c + 11392);
    const uint32_t hdr = lds32(c + 11400), cnt = lds32(c + 11404);
    const uint4 qm = lds128(c + 11408);
    const uint32_t rb = lds8(c + 11264 + r);
    uint4 lo[4];
    uint32_t cw[6];
#pragma unroll
    for (int j = 0; j < 4; ++j) lo[j] = lds128(c + (j * 128u + r) * 16u);
#pragma unroll
    for (int m = 0; m < 6; ++m) cw[m] = lds32(c + 8192u + (m * 128u + r) * 4u);
    const uint32_t lane = threadIdx.x & 31u, q = r >> 5;
    const uint32_t n_hard = cnt & 0xffu, n_rec = (cnt >> 8) & 0xffu;
    // this row's unit record: rows with records are counted in row order
    const uint32_t qmask = q == 0 ? qm.x : q == 1 ? qm.y : q == 2 ? qm.z : qm.w;
    const uint32_t base = (q > 0 ? __popc(qm.x) : 0) + (q > 1 ? __popc(qm.y) : 0) + (q > 2 ? __popc(qm.z) : 0);
#ifndef MLT_DIAG_C4_RECNOLOAD
    const uint32_t rec = (qmask >> lane) & 1u ? lds32(c + 11424u + 4u * (base + __popc(qmask & ((1u << lane) - 1u))))
                                               : 0u;
#else
    const uint32_t rec = (qmask >> lane) & 1u ? (qmask ^ base) : 0u;
#endif
    // hard escapes of this warp's quarter
    const uint32_t hb0 = q ? (hdr >> (8 * q)) & 0xffu : 0u, hb1 = q < 3 ? (hdr >> (8 * (q + 1))) & 0xffu : n_hard;
    const uint32_t h0 = c + 11424u + 4u * n_rec;
    esc.n = hb1 - hb0;
    esc.e0 = lane < esc.n ? lds32(h0 + 4u * (hb0 + lane)) : 0u;
    esc.e1 = lane + 32u < esc.n ? lds32(h0 + 4u * (hb0 + 32u + lane)) : 0u;
    // slot 7: the row's byte, or in flagged units of row half h the record's byte X_h
    const uint32_t t1 = prmt(T.y, rb, 0x4210u), t1x0 = prmt(T.y, rec >> 16, 0x4210u),
                   t1x1 = prmt(T.y, rec >> 24, 0x4210u);
    if (hdr & 0xffu)
        expand_row_c4<true>(lo, cw, T.x, t1, t1x0, t1x1, rec, o);
    else
        expand_row_c4<false>(lo, cw, T.x, t1, t1x0, t1x1, rec, o);
}

template <int G>
__device__ __forceinline__ void patch8_c4(uint32_t (&o)[32], uint32_t j, uint32_t v, uint32_t sel) {
#pragma unroll
    for (uint32_t x = 0; x < 8; ++x)
        if (x == j) o[8 * G + x] = prmt(o[8 * G + x], v, sel);
}

__device__ __forceinline__ void patch_hard_c4(uint32_t (&o)[32], uint32_t r, const EscC4& esc) {
    for (uint32_t e = 0; e < esc.n; ++e) {
        const uint32_t x0 = __shfl_sync(0xffffffffu, esc.e0, e & 31u), x1 = __shfl_sync(0xffffffffu, esc.e1, e & 31u);
        const uint32_t ent = e < 32u ? x0 : x1, idx = ent & 0xffffu;
        if (((idx >> 4) & 127u) == r) {
            // column k / 2 = 8 * (i >> 11) + (i & 15) / 2: the 16-k chunk picks
            // one of 4 groups of 8 registers, then 8 predicated selects
            const uint32_t j = (idx & 15u) >> 1, v = ent >> 16, sel = (idx & 1u) ? 0x5410u : 0x3254u;
            const uint32_t g = idx >> 11;
            if (g == 0) patch8_c4<0>(o, j, v, sel);
            else if (g == 1) patch8_c4<1>(o, j, v, sel);
            else if (g == 2) patch8_c4<2>(o, j, v, sel);
            else patch8_c4<3>(o, j, v, sel);
        }
    }
}

// raw fallback tile (16 KiB SWIZZLE_128B image): row r's logical 16-byte
// chunk q sits at chunk position q ^ (r % 8) of its 128-byte line
__device__ __forceinline__ void raw_row_ts(uint32_t sa, uint32_t r, uint32_t (&o)[32]) {
    const uint32_t base = sa + (r >> 3) * 1024u + (r & 7u) * 128u;
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
        const uint4 v = lds128(base + ((q ^ (r & 7u)) << 4));
        o[4 * q] = v.x, o[4 * q + 1] = v.y, o[4 * q + 2] = v.z, o[4 * q + 3] = v.w;
    }
}
// ---- codec 3 roles: three decoupled rings ---------------------------------
// (1) encoded-A ring in smem (A3 slots of 12432 B, 16 KiB when the GEMM has
//     raw fallback blocks): warp 0 streams every weight tile of the CTA's
//     task list into it, gated only by its decoders having READ the slot;
// (2) TMEM A slots (32 columns per tile): decoders -> MMA;
// (3) token-tile (B) ring in smem: warp 14 streams one B tile per k-block,
//     freed by the MMA's commit.
// Weight tile t of the CTA (all tasks, k-blocks, matrices in order) uses A
// slot t % A3 and TMEM slot t % T3, and is decoded by group t % kTsGroups
// (warps 6 + 4g .. 9 + 4g; A3 and T3 are multiples of kTsGroups).  The HBM
// stream is thus bounded by the smem ring depth and decoder speed, not by MMA
// completion as in a shared per-stage ring.
struct Ring3 {
    int a_slots, t_slots, b_slots, a_slot_bytes, b_bytes;
    uint8_t* a_ring;
    uint8_t* b_ring;
};

__device__ __forceinline__ void producer_a_ts(const GemmArgs& a, const Ring3& R, Smem* ctl, int n_virtual, int KB) {
    const uint64_t pol_w = l2_evict_first();
    int s = 0, t = 0;
    uint32_t ph = 0;
    for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
        const VTask tk = vtask(a, v, KB);
        const int rows = a.b_cnt ? a.b_cnt[tk.g] : a.rows_dense;
        if (rows <= 0) continue;
        const uint8_t* ab[kMaxMats];
        int tile_b[kMaxMats];
        for (int mt = 0; mt < a.n_mats; ++mt) {
            bool raw;
            ab[mt] = untag(a.a_table[(static_cast<int64_t>(mt) * a.G + tk.g) * a.RB + tk.rb], raw);
            tile_b[mt] = raw ? kATileBytes : enc_tile_bytes(a);
        }
        for (int n0 = tk.c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap)
            for (int kb = tk.kb0; kb < tk.kb1; ++kb)
                for (int mt = 0; mt < a.n_mats; ++mt, ++t) {
                    mbar_wait(&ctl->empty[s], ph ^ 1);
                    if (a.ktrace && blockIdx.x == 0 && t < 256) a.ktrace[t] = globaltimer();
                    mbar_expect_tx(&ctl->full[s], tile_b[mt]);
                    bulk_g2s(R.a_ring + s * R.a_slot_bytes, ab[mt] + static_cast<int64_t>(kb) * tile_b[mt],
                             tile_b[mt], &ctl->full[s], pol_w);
                    if (++s == R.a_slots) { s = 0; ph ^= 1; }
                }
    }
}

__device__ __forceinline__ void producer_b_ts(const GemmArgs& a, const Ring3& R, Smem* ctl, int n_virtual, int KB) {
    const uint64_t pol_x = l2_evict_last();
    int s = 0;
    uint32_t ph = 0;
    for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
        const VTask tk = vtask(a, v, KB);
        const int rows = a.b_cnt ? a.b_cnt[tk.g] : a.rows_dense;
        if (rows <= 0) continue;
        const int row0 = a.b_off ? a.b_off[tk.g] : 0;
        for (int n0 = tk.c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
            const int ntp = (min(a.n_cap, rows - n0) + 15) & ~15;
            for (int kb = tk.kb0; kb < tk.kb1; ++kb) {
                mbar_wait(&ctl->bempty[s], ph ^ 1);
                mbar_expect_tx(&ctl->bfull[s], ntp * 128);
                bulk_g2s(R.b_ring + s * R.b_bytes,
                         a.b + static_cast<int64_t>(kb) * a.R * 128 + static_cast<int64_t>(row0 + n0) * 128, ntp * 128,
                         &ctl->bfull[s], pol_x);
                if (++s == R.b_slots) { s = 0; ph ^= 1; }
            }
        }
    }
}

// Decoder warps 6-13: warp w decodes rows 32 (w % 4) .. +31 (its TMEM lane
// quarter) of every tile t with t % 2 == (w - 6) / 4: smem -> registers ->
// release the A slot (one arrival per warp) -> wait for the TMEM slot ->
// tcgen05.st -> wait::st -> one arrival per warp on the slot's dfull.
template <int kMode>
__device__ __forceinline__ void decoder_role_ts(const GemmArgs& a, const Ring3& R, Smem* ctl, int n_virtual, int KB,
                                                uint32_t tmem) {
    const int w = static_cast<int>(threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    constexpr int kTsGroups = ts_groups(kMode);
    const int grp = (w - 6) >> 2;    // tile t is decoded by group t % kTsGroups
    const uint32_t q = static_cast<uint32_t>(w) & 3u;  // TMEM lane quarter
    const uint32_t r = q * 32u + lane;
    const uint32_t tl = tmem + ((q * 32u) << 16) + static_cast<uint32_t>(a.acc_stages * a.n_mats * a.n_cap);
    int t = 0, s = 0, ts = 0, tg = 0;  // tile counter, its A slot, TMEM slot and decoder group
    uint32_t ph = 0, tph = 0;        // ring phases
    for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
        const VTask tk = vtask(a, v, KB);
        const int rows = a.b_cnt ? a.b_cnt[tk.g] : a.rows_dense;
        if (rows <= 0) continue;
        bool raw0 = false, raw1 = false;
        untag(a.a_table[static_cast<int64_t>(tk.g) * a.RB + tk.rb], raw0);
        if (a.n_mats == 2) untag(a.a_table[(static_cast<int64_t>(a.G) + tk.g) * a.RB + tk.rb], raw1);
        for (int n0 = tk.c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap)
            for (int kb = tk.kb0; kb < tk.kb1; ++kb)
                for (int mt = 0; mt < a.n_mats; ++mt) {
                    if (tg == grp) {
                        // CTA-0 trace (warp of lane quarter 0): rows 1-4 = landed, decoded, slot granted, stored
                        unsigned long long* const kt =
                            (a.ktrace && blockIdx.x == 0 && t < 256 && q == 0 && lane == 0) ? a.ktrace + t : nullptr;
                        mbar_wait(&ctl->full[s], ph);
                        if (kt) kt[256] = globaltimer();
                        const uint32_t sa = smem_u32(R.a_ring + s * R.a_slot_bytes);
                        uint32_t o[32];
                        EscC4 esc{0u, 0u, 0u};
                        if (mt ? raw1 : raw0) {
                            raw_row_ts(sa, r, o);
                        } else if constexpr (kMode == 4) {
                            decode_row_c4(sa, r, o, esc);
#ifndef MLT_DIAG_C4_NOHARD  // diagnostic builds (tools/diag_build.sh) only
                            if (esc.n) patch_hard_c4(o, r, esc);
#endif
                        } else {
                            decode_row_ts(sa, r, o);
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&ctl->empty[s]);
                        if (kt) kt[512] = globaltimer();
                        mbar_wait(&ctl->aslot_empty[ts], tph ^ 1);
                        if (kt) kt[768] = globaltimer();
                        tc_fence_after();
                        tmem_st32(tl + static_cast<uint32_t>(ts * 32), o);
                        tmem_wait_st();


                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&ctl->dfull[ts]);
                        if (kt) kt[1024] = globaltimer();
                    }
                    ++t;
                    if (++tg == kTsGroups) tg = 0;
                    if (++s == R.a_slots) { s = 0; ph ^= 1; }
                    if (++ts == R.t_slots) { ts = 0; tph ^= 1; }
                }
    }
}

// MMA warp (lane 0 issues): per k-block wait its B tile, per matrix wait the
// decoded TMEM A slot, 4 x (M128 N ntp K16) with A from TMEM, commit the A
// slot; after the k-block commit the B slot; after the last k-block commit
// the accumulator stage to the epilogue.
__device__ __forceinline__ void mma_role_ts(const GemmArgs& a, const Ring3& R, Smem* ctl, int n_virtual, int KB,
                                            uint32_t tmem) {
    const uint32_t lane = threadIdx.x & 31u;
    const int acc_cols = a.n_mats * a.n_cap;
    const uint32_t ta0 = tmem + static_cast<uint32_t>(a.acc_stages * acc_cols);
    int ts = 0, sb = 0, acc = 0, t = 0;
    uint32_t tph = 0, bph = 0, acc_phase = 0;
    for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
        const VTask tk = vtask(a, v, KB);
        const int rows = a.b_cnt ? a.b_cnt[tk.g] : a.rows_dense;
        if (rows <= 0) continue;
        for (int n0 = tk.c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
            const int ntp = (min(a.n_cap, rows - n0) + 15) & ~15;
            const uint32_t idesc = idesc_bf16(128, ntp);
            mbar_wait(&ctl->tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d0 = tmem + acc * acc_cols;
            for (int kb = tk.kb0; kb < tk.kb1; ++kb) {
                // the k-block's B tile and its n_mats decoded A tiles (TMEM slots ts, ts+1 mod t_slots)
                mbar_wait(&ctl->bfull[sb], bph);
                int ts1 = ts + 1;
                uint32_t tph1 = tph;
                if (ts1 == R.t_slots) { ts1 = 0; tph1 ^= 1; }
                mbar_wait(&ctl->dfull[ts], tph);
                if (a.ktrace && blockIdx.x == 0 && t < 256 && lane == 0) a.ktrace[1280 + t] = globaltimer();
                if (a.n_mats == 2) mbar_wait(&ctl->dfull[ts1], tph1);
                tc_fence_after();
                if (elect_one()) {  // warp-uniform operands: no per-MMA register -> uniform moves
                    const uint32_t bs = smem_u32(R.b_ring + sb * R.b_bytes);
                    const uint32_t a0 = ta0 + ts * 32, a1 = ta0 + ts1 * 32;
#pragma unroll
                    for (int k = 0; k < kBlockK / 16; ++k) {
                        const uint64_t bd = sdesc_sw128(bs + k * 32);
                        const uint32_t accf = (kb != tk.kb0 || k != 0) ? 1u : 0u;
                        umma_bf16_ts(d0, a0 + k * 8, bd, idesc, accf);
                        if (a.n_mats == 2) umma_bf16_ts(d0 + a.n_cap, a1 + k * 8, bd, idesc, accf);
                    }
                    umma_commit(&ctl->aslot_empty[ts]);
                    if (a.n_mats == 2) umma_commit(&ctl->aslot_empty[ts1]);
                    umma_commit(&ctl->bempty[sb]);
                    if (kb + 1 == tk.kb1) umma_commit(&ctl->tfull[acc]);
                }
                __syncwarp();
                t += a.n_mats;
                if (a.n_mats == 2) {
                    ts = ts1 + 1, tph = tph1;
                    if (ts == R.t_slots) { ts = 0; tph ^= 1; }
                } else {
                    ts = ts1, tph = tph1;
                }
                if (++sb == R.b_slots) { sb = 0; bph ^= 1; }
            }
            if (++acc == a.acc_stages) { acc = 0; acc_phase ^= 1; }
        }
    }
}

// kMode: 0 = raw / codec 1 (shared-stage ring), 3 / 4 = the TMEM-operand
// engine with the 4-bit / 3-bit decoder (one decoder per kernel keeps the
// decoder warps' hot loop small: codec 4 with both decoders and its escape
// sweep in one kernel stalled on instruction fetch, ncu no_instruction 8.7
// per issue vs 0.4)
template <int kMode>
__global__ void __launch_bounds__(kMode ? ts_threads(kMode) : kThreadsCodec, 1) gemm_tc_kernel(const GemmArgs a) {
    constexpr bool kTs = kMode != 0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KiB alignment for the SWIZZLE_128B atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    const int a_bytes = a.n_mats * kATileBytes;  // A slots of one k-block
    const int b_bytes = a.n_cap * 128;            // B tile of one k-block
    const int kps = a.kps;                        // k-blocks per ring stage (1, or 2 for codec n_mats = 1)
    // stage = [kps x A tiles (16 KiB slots) | kps x B tile]; with the codec
    // the encoded A tiles land at the end of their slots and are decoded in
    // place; tile t of a stage (t = j * n_mats + mt) sits at t * 16 KiB
    const int stage_bytes = kps * (a_bytes + b_bytes);
    const int stages = a.stages;
    // codec 3: [A ring: stages x a3_slot_bytes][B ring: b3_slots x b_bytes][ctl]
    // (the B ring's SWIZZLE_128B atoms need 1 KiB alignment)
    Ring3 R3{stages, a.t3_slots, a.b3_slots, a.a3_slot_bytes, b_bytes, smem,
             smem + ((stages * a.a3_slot_bytes + 1023) & ~1023)};
    Smem* ctl = reinterpret_cast<Smem*>(kTs ? R3.b_ring + a.b3_slots * b_bytes : smem + stages * stage_bytes);

    const uint32_t warp = warp_idx_sync();
    const uint32_t lane = threadIdx.x & 31;

    unsigned long long* const tr = a.trace ? a.trace + blockIdx.x * 8 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = globaltimer();
    const int acc_cols = a.n_mats * a.n_cap;     // TMEM columns per accumulator stage
    const int acc_stages = a.acc_stages;          // 1 or 2

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&ctl->full[s], 1);
            mbar_init(&ctl->empty[s], 1);
        }
        for (int s = 0; s < acc_stages; ++s) {
            mbar_init(&ctl->tfull[s], 1);
            mbar_init(&ctl->tempty[s], 4);
        }
        if (a.codec == 1)
            for (int s = 0; s < stages; ++s) mbar_init(&ctl->dfull[s], 1);
        if (kTs) {  // A slots are read / written by the 4 warps of one decoder group
            for (int s = 0; s < stages; ++s) mbar_init(&ctl->empty[s], 4);
            for (int s = 0; s < a.t3_slots; ++s) {
                mbar_init(&ctl->dfull[s], 4);
                mbar_init(&ctl->aslot_empty[s], 1);
            }
            for (int s = 0; s < a.b3_slots; ++s) {
                mbar_init(&ctl->bfull[s], 1);
                mbar_init(&ctl->bempty[s], 1);
            }
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&ctl->tmem_base, a.tmem_cols);
    pdl_trigger();
    if (warp == 0 && lane == 0 && static_cast<int>(blockIdx.x) < a.G * a.RB * a.n_chunks * a.k_splits) {
        // immutable weights: warm L2 with this CTA's first A tiles while the
        // predecessor kernel drains (PDL); activations only after the wait
        const int u = static_cast<int>(blockIdx.x) / a.k_splits, ks = static_cast<int>(blockIdx.x) % a.k_splits;
        const int g = (u / a.n_chunks) % a.G, rb = u / a.n_chunks / a.G;
        const int KBt = a.K / kBlockK, kb0 = ks * KBt / a.k_splits;
        const int nkb = min(4, (ks + 1) * KBt / a.k_splits - kb0);
        for (int mt = 0; mt < a.n_mats; ++mt) {
            bool raw;
            const uint8_t* p = untag(a.a_table[(static_cast<int64_t>(mt) * a.G + g) * a.RB + rb], raw);
            const int tile = (a.codec && !raw) ? enc_tile_bytes(a) : kATileBytes;
            prefetch_l2(p + static_cast<int64_t>(kb0) * tile, static_cast<uint32_t>(nkb * tile));
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    // in-kernel timing starts once the predecessor is done (with PDL the CTA
    // may have been resident, prefetching weights, while it drained)
    if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[0], globaltimer());
    const uint32_t tmem = ctl->tmem_base;
    if (tr && threadIdx.x == 0) tr[1] = globaltimer();

    // virtual tile = (row block, group, N-chunk, K-split), K-split fastest
    const int n_virtual = a.sk_parts ? a.sk_full + a.sk_tail * a.sk_parts : a.G * a.RB * a.n_chunks * a.k_splits;
    const int KB = a.K / kBlockK;

    if (kTs && (warp < 2 || warp >= 6)) {
        // ===== codec 3: decoupled rings (the epilogue below is shared) =====
        if (warp == 0) {
            if (lane == 0) producer_a_ts(a, R3, ctl, n_virtual, KB);
        } else if (warp == ts_bwarp(kMode)) {
            if (lane == 0) producer_b_ts(a, R3, ctl, n_virtual, KB);
        } else if (warp == 1) {
            mma_role_ts(a, R3, ctl, n_virtual, KB, tmem);
        } else {
            decoder_role_ts<kMode>(a, R3, ctl, n_virtual, KB, tmem);
        }
    } else if (warp == 0) {
        // ===== producer =====
        if (elect_one()) {
            const uint64_t pol_w = l2_evict_first(), pol_x = l2_evict_last();
            int stage = 0, kstep = 0;
            uint32_t phase = 0;
            for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
                const VTask tk = vtask(a, v, KB);
                const int c = tk.c, g = tk.g, rb = tk.rb, kb0 = tk.kb0, kb1 = tk.kb1;
                const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
                if (rows <= 0) continue;
                const int row0 = a.b_off ? a.b_off[g] : 0;
                const uint8_t* ab[kMaxMats];
                int tile_b[kMaxMats], slot_off[kMaxMats], tx = 0;  // per matrix: stored tile bytes, offset in slot
                for (int mt = 0; mt < a.n_mats; ++mt) {
                    bool raw;
                    ab[mt] = untag(a.a_table[(static_cast<int64_t>(mt) * a.G + g) * a.RB + rb], raw);
                    tile_b[mt] = (a.codec && !raw) ? kCodecTile : kATileBytes;
                    slot_off[mt] = (a.codec && !raw) ? kCodecOff : 0;
                    tx += tile_b[mt];
                }
                for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                    const int nt = min(a.n_cap, rows - n0);
                    const int ntp = (nt + 15) & ~15;
                    for (int kb = kb0; kb < kb1; kb += kps) {
                        const int nk = min(kps, kb1 - kb);
                        mbar_wait(&ctl->empty[stage], phase ^ 1);
                        if (a.ktrace && blockIdx.x == 0 && kstep < 256) a.ktrace[kstep] = globaltimer();
                        ++kstep;
                        uint8_t* const st = smem + stage * stage_bytes;
                        uint8_t* sb = st + kps * a_bytes;
                        if (tr && v == static_cast<int>(blockIdx.x) && kb == kb0 && n0 == c * a.n_cap)
                            tr[2] = globaltimer();
                        mbar_expect_tx(&ctl->full[stage], nk * (tx + ntp * 128));
                        for (int j = 0; j < nk; ++j) {
                            for (int mt = 0; mt < a.n_mats; ++mt)
                                bulk_g2s(st + (j * a.n_mats + mt) * kATileBytes + slot_off[mt],
                                         ab[mt] + static_cast<int64_t>(kb + j) * tile_b[mt], tile_b[mt],
                                         &ctl->full[stage], pol_w);
                            const uint8_t* src = a.b + static_cast<int64_t>(kb + j) * a.R * 128 +
                                                 static_cast<int64_t>(row0 + n0) * 128;
                            bulk_g2s(sb + j * b_bytes, src, ntp * 128, &ctl->full[stage], pol_x);
                        }
                        if (++stage == stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0, kstep = 0;
        uint32_t acc_phase = 0;
        for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
            const VTask tk = vtask(a, v, KB);
            const int c = tk.c, g = tk.g, kb0 = tk.kb0, kb1 = tk.kb1;
            const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
            if (rows <= 0) continue;
            for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                const int nt = min(a.n_cap, rows - n0);
                const int ntp = (nt + 15) & ~15;
                const uint32_t idesc = idesc_bf16(128, ntp);
                mbar_wait(&ctl->tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d0 = tmem + acc * acc_cols;
                for (int kb = kb0; kb < kb1; kb += kps) {
                    const int nk = min(kps, kb1 - kb);
                    mbar_wait(&ctl->full[stage], phase);
                    if (a.codec) mbar_wait(&ctl->dfull[stage], phase);
                    tc_fence_after();
                    if (a.ktrace && blockIdx.x == 0 && kstep < 256 && lane == 0) a.ktrace[768 + kstep] = globaltimer();
                    ++kstep;
                    if (tr && lane == 0 && v == static_cast<int>(blockIdx.x) && kb == kb0 && n0 == c * a.n_cap)
                        tr[3] = globaltimer();
                    if (elect_one()) {
                        const uint32_t st = smem_u32(smem + stage * stage_bytes);
                        for (int j = 0; j < nk; ++j) {
                            const uint32_t sa = st + j * a_bytes;
                            const uint32_t sb = st + kps * a_bytes + j * b_bytes;
#pragma unroll
                            for (int k = 0; k < kBlockK / 16; ++k) {
                                const uint64_t bd = sdesc_sw128(sb + k * 32);
                                for (int mt = 0; mt < a.n_mats; ++mt)
                                    umma_bf16(d0 + mt * a.n_cap, sdesc_sw128(sa + mt * kATileBytes + k * 32),
                                              bd, idesc, (kb + j != kb0 || k != 0) ? 1u : 0u);
                            }
                        }
                        umma_commit(&ctl->empty[stage]);
                        if (kb + nk >= kb1) umma_commit(&ctl->tfull[acc]);
                    }
                    __syncwarp();
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
                if (++acc == acc_stages) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= 6) {
        // ===== decoders (codec): encoded tiles -> bf16 smem images, in place =====
        if (a.dec_groups == 1)
            decoder_role<256>(a, smem, ctl, stages, stage_bytes, kps, n_virtual, KB);
        else
            decoder_role<128>(a, smem, ctl, stages, stage_bytes, kps, n_virtual, KB);
    } else {
        // ===== epilogue: TMEM -> registers -> global =====
        const uint32_t quarter = warp & 3;  // TMEM lanes this warp may access
        float* const scr = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ctl) + kCtlBytes) + quarter * 512;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int v = blockIdx.x; v < n_virtual; v += gridDim.x) {
            const VTask tk = vtask(a, v, KB);
            const int ks = tk.part >= 0 ? 0 : v % a.k_splits;
            const int c = tk.c, g = tk.g, rb = tk.rb;
            const int rows = a.b_cnt ? a.b_cnt[g] : a.rows_dense;
            if (rows <= 0) continue;
            const int row0 = a.b_off ? a.b_off[g] : 0;
            const int mbase = rb * kBlockM + quarter * 32;  // this warp's 32 output features
            // K-split partials go to separate buffers, reduced by the consumer
            float* const outp = a.out_f32 ? a.out_f32 + static_cast<int64_t>(ks) * a.split_stride : nullptr;
            const float* const resid = a.k_splits == 1 ? a.residual : nullptr;
            for (int n0 = c * a.n_cap; n0 < rows; n0 += a.n_chunks * a.n_cap) {
                const int nt = min(a.n_cap, rows - n0);
                mbar_wait(&ctl->tfull[acc], acc_phase);
                tc_fence_after();
                if (tr && warp == 2 && lane == 0 && v == static_cast<int>(blockIdx.x) && n0 == c * a.n_cap)
                    tr[5] = globaltimer();
                const uint32_t t0 = tmem + ((quarter * 32u) << 16) + acc * acc_cols;
                // Each 32-feature x 16-token chunk goes TMEM -> registers ->
                // a per-warp smem transpose -> 16-byte global stores along the
                // feature axis (row-contiguous in the output), instead of 16
                // scalar stores per thread (6x slower, tools/trace_gemm.py).
                for (int c2 = 0; c2 < nt; c2 += 16 * kEpiChunks) {
                    // issue the TMEM loads of two 16-token chunks (both matrices
                    // for SiLU), then a single wait: one TMEM round trip per 32 tokens
                    const bool two = kEpiChunks == 2 && c2 + 16 < nt;
                    uint32_t r0[2][16], r1[2][16];
                    tmem_ld16_async(t0 + c2, r0[0]);
                    if (two) tmem_ld16_async(t0 + c2 + 16, r0[1]);
                    if (a.epi != kEpiF32) {
                        tmem_ld16_async(t0 + a.n_cap + c2, r1[0]);
                        if (two) tmem_ld16_async(t0 + a.n_cap + c2 + 16, r1[1]);
                    }
                    tmem_wait_ld();
                    tmem_regs_ready(r0[0]);
                    if (two) tmem_regs_ready(r0[1]);
                    if (a.epi != kEpiF32) {
                        tmem_regs_ready(r1[0]);
                        if (two) tmem_regs_ready(r1[1]);
                    }
#pragma unroll
                    for (int h = 0; h < kEpiChunks; ++h) {
                        const int c = c2 + 16 * h;
                        if (c >= nt) break;
                        if (a.epi == kEpiF32) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) scr[j * 32 + lane] = __uint_as_float(r0[h][j]) * a.alpha;
                            __syncwarp();
                            const int f = (lane & 7) * 4;
                            float4 rv[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {  // residual loads first (all in flight)
                                const int j = q * 4 + (lane >> 3);
                                rv[q] = (resid && c + j < nt)
                                            ? *reinterpret_cast<const float4*>(
                                                  resid + (row0 + n0 + c + j) * static_cast<int64_t>(a.ldr) + mbase + f)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int j = q * 4 + (lane >> 3);
                                if (c + j < nt) {
                                    float4 v = *reinterpret_cast<const float4*>(scr + j * 32 + f);
                                    v.x += rv[q].x; v.y += rv[q].y; v.z += rv[q].z; v.w += rv[q].w;
                                    *reinterpret_cast<float4*>(
                                        outp + (row0 + n0 + c + j) * static_cast<int64_t>(a.ldo) + mbase + f) = v;
                                }
                            }
                            __syncwarp();
                        } else if (tk.part >= 0) {  // stream-K part: fp32 g and u to the scratch
                            float* const pb = a.sk_scratch + static_cast<int64_t>(tk.tile * a.sk_parts + tk.part) *
                                                                 a.n_mats * a.sk_rows * 128;
#pragma unroll
                            for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    scr[j * 32 + lane] = __uint_as_float(mt ? r1[h][j] : r0[h][j]);
                                __syncwarp();
                                const int f = (lane & 7) * 4;
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const int j = q * 4 + (lane >> 3);
                                    if (c + j < nt)
                                        *reinterpret_cast<float4*>(
                                            pb + (static_cast<int64_t>(mt) * a.sk_rows + n0 + c + j) * 128 + quarter * 32 + f) =
                                            *reinterpret_cast<const float4*>(scr + j * 32 + f);
                                }
                                __syncwarp();
                            }
                        } else {  // kEpiSiluPacked
                            uint16_t* sb = reinterpret_cast<uint16_t*>(scr);
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                sb[j * 32 + lane] =
                                    f32_to_bf16_bits(silu(__uint_as_float(r0[h][j])) * __uint_as_float(r1[h][j]));
                            __syncwarp();
                            const int f = (lane & 3) * 8;
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
                                const int j = q * 8 + (lane >> 2);
                                if (c + j < nt)
                                    *reinterpret_cast<uint4*>(a.out_packed + b_packed_off(row0 + n0 + c + j, mbase + f,
                                                                                          a.out_R)) =
                                        *reinterpret_cast<const uint4*>(sb + j * 32 + f);
                            }
                            __syncwarp();
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&ctl->tempty[acc]);
                if (++acc == acc_stages) { acc = 0; acc_phase ^= 1; }
            }
            if (tk.part >= 0) {
                // arrive, wait for the tile's other parts (monotonic counter:
                // this launch's target is the next multiple of sk_parts), then
                // finish rows [part*rows/S, (part+1)*rows/S): every part summed
                // in part order (deterministic), SiLU, packed bf16
                __threadfence();
                asm volatile("bar.sync 4, 128;" ::: "memory");  // the 4 epilogue warps' stores are fenced
                if (warp == 2 && lane == 0) {
                    // 64-bit monotonic counter: never wraps (2^64 / S launches)
                    const unsigned long long S = static_cast<unsigned long long>(a.sk_parts);
                    const unsigned long long old = atomicAdd(a.sk_count + tk.tile, 1ull);
                    const unsigned long long target = (old / S + 1) * S;
                    const unsigned long long t_start = globaltimer();
                    while (ld_acquire(a.sk_count + tk.tile) < target) {
                        __nanosleep(64);
                        if (globaltimer() - t_start > kSpinLimitNs) __trap();
                    }
                }
                asm volatile("bar.sync 4, 128;" ::: "memory");
                __threadfence();
                const int S = a.sk_parts;
                const int r0s = tk.part * rows / S, r1s = (tk.part + 1) * rows / S;
                const float* sb = a.sk_scratch + static_cast<int64_t>(tk.tile) * S * a.n_mats * a.sk_rows * 128 +
                                  quarter * 32 + lane;
                const int64_t pstride = static_cast<int64_t>(a.n_mats) * a.sk_rows * 128;
                uint16_t* st16 = reinterpret_cast<uint16_t*>(scr);
                for (int r = r0s; r < r1s; ++r) {
                    float gs = 0.f, us = 0.f;
                    constexpr int kB = 8;  // loads in flight before the ordered sums
                    for (int p0 = 0; p0 < S; p0 += kB) {
                        float gv[kB], uv[kB];
#pragma unroll
                        for (int q = 0; q < kB; ++q) {
                            const float* bp = sb + (p0 + q) * pstride + static_cast<int64_t>(r) * 128;
                            gv[q] = p0 + q < S ? __ldcg(bp) : 0.f;
                            uv[q] = p0 + q < S ? __ldcg(bp + static_cast<int64_t>(a.sk_rows) * 128) : 0.f;
                        }
#pragma unroll
                        for (int q = 0; q < kB; ++q)
                            if (p0 + q < S) gs += gv[q], us += uv[q];
                    }
                    st16[lane] = f32_to_bf16_bits(silu(gs) * us);
                    __syncwarp();
                    if (lane < 4)
                        *reinterpret_cast<uint4*>(a.out_packed + b_packed_off(row0 + r, mbase + 8 * lane, a.out_R)) =
                            *reinterpret_cast<const uint4*>(st16 + 8 * lane);
                    __syncwarp();
                }
            }
        }
    }
    if (tr && warp == 1 && lane == 0) tr[4] = globaltimer();  // all MMAs issued
    if (tr && warp == 2 && lane == 0) tr[6] = globaltimer();  // this warp's epilogue done
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, a.tmem_cols);
    }
    if (tr && threadIdx.x == 0) tr[7] = globaltimer();
    if (a.timing && threadIdx.x == 0) atomicMin(&a.timing[1], ~globaltimer());
}

}  // namespace

int gemm_smem_bytes(int n_mats, int n_cap, int stages, int kps) {
    return stages * kps * (n_mats * kATileBytes + n_cap * 128) +
           1024 /*align*/ + kCtlBytes + kEpiScratch;
}

cudaError_t launch_gemm(GemmArgs a, int num_sms, cudaStream_t stream) {
    if (a.codec == 2) return launch_gemm_codec(a, num_sms, stream);
    if (a.n_mats < 1 || a.n_mats > kMaxMats || a.K % kBlockK || a.n_cap % 16 || a.n_cap < 16 ||
        a.n_cap > 256 || a.R % 16 || a.n_chunks < 1 || a.k_splits < 1 ||
        a.k_splits > a.K / kBlockK || (a.k_splits > 1 && a.epi != kEpiF32) ||
        (a.epi == kEpiF32 && (a.ldo % 4 || a.ldr % 4 || a.split_stride % 4)))  // 16-byte epilogue stores
        return cudaErrorInvalidValue;
    // codec with one matrix: two k-blocks per ring stage, so each stage's
    // fixed decode cost (barriers, proxy fence, dfull round trip) covers two
    // encoded tiles, as it does for the two matrices of gate/up
    // (only while that still leaves >= 4 stages: mu = 256 down, n_cap 128, would get 2)
    // codec 3 keeps A slots in TMEM next to the accumulators: at most 256
    // accumulator columns (a wide prefill tile loops over more token chunks)
    if (a.codec >= 3 && a.n_mats * a.n_cap > 256) a.n_cap = 256 / a.n_mats;
    const int budget = 227 * 1024 - 1024 - kCtlBytes - kEpiScratch;
    a.kps = (a.codec && a.n_mats == 1 && budget / (2 * (kATileBytes + a.n_cap * 128)) >= 4) ? 2 : 1;
    const int per_stage = a.kps * (a.n_mats * kATileBytes + a.n_cap * 128);
    a.stages = budget / per_stage;
    if (a.stages > 8) a.stages = 8;
    if (a.codec == 1) {
        if (a.dec_groups < 1 || a.dec_groups > kMaxDecGroups) return cudaErrorInvalidValue;
        a.stages -= a.stages % a.dec_groups;  // decoder groups own whole stages
    }
    if (a.codec < 0 || a.codec > 4) return cudaErrorInvalidValue;  // 2 dispatched above
    const int acc_cols = a.n_mats * a.n_cap;
    a.acc_stages = (2 * acc_cols <= 512) ? 2 : 1;
    int need = a.acc_stages * acc_cols;
    if (a.codec >= 3) {
        // decoupled rings (Ring3): token tiles (3-4 slots), encoded A slots
        // (12432 B, or 16 KiB when raw fallback blocks may appear) in the rest
        // of smem, TMEM A slots (32 columns per tile) next to the accumulators
        a.kps = 1;
        a.b3_slots = a.n_cap * 128 <= 16384 ? 4 : 3;
        if (a.codec == 4 && (a.enc_tile % 16 || a.enc_tile < 0 || a.enc_tile > kATileBytes || (a.enc_tile && a.enc_tile < 11424)))
            return cudaErrorInvalidValue;
        a.a3_slot_bytes = a.codec_raw ? kATileBytes : enc_tile_bytes(a);
        a.stages = std::min(kMaxRing, (budget - 1024 - a.b3_slots * a.n_cap * 128) / a.a3_slot_bytes);
        if ((512 - need) / 32 < 4 && a.acc_stages == 2) {
            a.acc_stages = 1;
            need = acc_cols;
        }
        a.t3_slots = std::min(kMaxRing, (512 - need) / 32);
        // tile t goes to decoder group t % kTsGroups, so both rings' slot counts
        // are multiples of the group count: every slot then belongs to one group,
        // which meets it phase after phase (a group skipping a phase of a slot it
        // shares could pass a parity wait one phase early: mbarrier parity aliases)
        const int groups = ts_groups(a.codec);
        a.stages -= a.stages % groups;
        a.t3_slots -= a.t3_slots % groups;
        if (a.t3_slots < groups || a.stages < groups) return cudaErrorInvalidValue;
        need += a.t3_slots * 32;
    }
    if (a.stages < 2) return cudaErrorInvalidValue;
    int cols = 32;
    while (cols < need) cols <<= 1;
    a.tmem_cols = cols;
    const int smem = a.codec >= 3 ? ((a.stages * a.a3_slot_bytes + 1023) & ~1023) + a.b3_slots * a.n_cap * 128 +
                                        1024 + kCtlBytes + kEpiScratch
                                  : gemm_smem_bytes(a.n_mats, a.n_cap, a.stages, a.kps);
    void (*const kern)(const GemmArgs) = a.codec == 4   ? gemm_tc_kernel<4>
                                         : a.codec == 3 ? gemm_tc_kernel<3>
                                                        : gemm_tc_kernel<0>;
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024); e != cudaSuccess)
        return e;
    a.sk_full = a.sk_tail = a.sk_parts = 0;
    if (a.sk_scratch && a.sk_count && a.sk_rows > 0 && a.epi == kEpiSiluPacked && a.n_mats == 2 &&
        a.k_splits == 1 && a.n_chunks == 1) {
        // stream-K tail: a partial last wave of `tail` tiles would leave
        // num_sms - tail SMs idle for one whole tile time
        const int nv = a.G * a.RB, tail = nv % num_sms;
        int S = tail > 0 ? num_sms / tail : 0;
        if (S > a.K / kBlockK / 2) S = a.K / kBlockK / 2;  // parts of >= 2 k-blocks
        if (nv > num_sms && S >= 2) {
            a.sk_full = nv - tail;
            a.sk_tail = tail;
            a.sk_parts = S;
        }
    }
    if (a.sk_parts) {
        // the tail's parts wait on each other: only with every CTA co-resident
        // (1 CTA per SM at this smem size; fewer SMs under MPS / green
        // contexts / a concurrent kernel) -> otherwise run without the tail
        // (cached per device and block size: the occupancy query costs host microseconds)
        static int cache[64][kMaxDecGroups + 3] = {};
        int dev = 0;
        const int slot = a.codec >= 3 ? kMaxDecGroups + a.codec - 2 : a.codec ? a.dec_groups : 0;
        int per_sm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
            if (!cache[dev][slot] &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cache[dev][slot], kern,
                                                              a.codec >= 3 ? ts_threads(a.codec)
                                                              : a.codec    ? kThreadsCodec
                                                                           : kThreadsRaw,
                                                              227 * 1024 - 1024) != cudaSuccess)
                cache[dev][slot] = 0;
            per_sm = cache[dev][slot];
        }
        if (per_sm < 1) a.sk_full = a.sk_tail = a.sk_parts = 0;
    }
    const int n_virtual = a.sk_parts ? a.sk_full + a.sk_tail * a.sk_parts : a.G * a.RB * a.n_chunks * a.k_splits;
    const int grid = n_virtual < num_sms ? n_virtual : num_sms;
    if (grid <= 0) return cudaSuccess;
    const dim3 block(a.codec >= 3 ? ts_threads(a.codec) : a.codec ? kThreadsCodec : kThreadsRaw);
    if (a.sk_parts) {
        // cooperative: the driver guarantees co-residency of the whole grid or
        // refuses the launch (then: the same GEMM without the stream-K tail)
        const cudaError_t e = launch_k_coop(kern, dim3(grid), block, smem, stream, a);
        if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported) return e;
        a.sk_full = a.sk_tail = a.sk_parts = 0;
        const int nv = a.G * a.RB * a.n_chunks * a.k_splits;
        return launch_k(kern, dim3(nv < num_sms ? nv : num_sms), block, smem, stream, a);
    }
    return launch_k(kern, dim3(grid), block, smem, stream, a);
}

}  // namespace mltk
