// kernels_tiny_impl.cuh -- the tiny-DFA kernel template (design notes: kernels_tiny.cu).
// Instantiated per (B, TMA) in kernels_tiny_inst_*.cu so the register-unrolled variants
// compile in parallel.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "kernels_common.cuh"

namespace parem {

namespace {

constexpr uint32_t kT = kTinyThreads;       // 512 threads per CTA, one CTA per SM
constexpr uint32_t kWarps = kT / 32;
constexpr uint32_t kRPL = 2;                // chunks (rows) per lane: two independent chains
constexpr uint32_t kRowsW = 32 * kRPL;      // rows per warp = rows of one TMA box
constexpr uint32_t kRows = kT * kRPL;       // chunks per CTA
constexpr uint32_t kBoxBytes = 64;          // TMA box: 64 rows x 64 bytes = 4 KB
constexpr uint32_t kStageBytes = kRowsW * kBoxBytes;
constexpr uint32_t kMaxStages = 3;

__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ __forceinline__ size_t al1k(size_t x) { return (x + 1023) & ~(size_t)1023; }

struct TinySmem {
    size_t tabk, tab1, lcnt, loff, llist, uni, mend, mhits, wend, whits, mbar, flag, total;
};

// Row strides of the per-lane dense maps in shared memory.  Lane l writes ITS row (all
// Qpad entries) while the warp's composition reads one row at the lanes' own states: with
// a plain Qpad stride the writes of 32 lanes hit the same banks (86.8 % of the store
// wavefronts conflicted, profiles/r01_ncu_full_cfg2_details.txt).  An odd word stride for
// the u32 hits (Qpad + 1) and a 5-word stride for the u8 ends make both patterns
// conflict-free (lane rows land on distinct banks; a read row spreads the lanes' states).
__host__ __device__ __forceinline__ uint32_t tiny_mend_stride(uint32_t Qpad) { return (Qpad < 4 ? 4u : Qpad) + 4u; }
__host__ __device__ __forceinline__ uint32_t tiny_mhits_stride(uint32_t Qpad) { return Qpad + 1u; }

// Offsets relative to a 1024-aligned base (the kernel aligns the dynamic smem pointer).
// `stages` = TMA stages per warp (0: no TMA staging).
__host__ __device__ __forceinline__ TinySmem tiny_layout(uint32_t Qp, uint32_t Qpad, uint32_t A, uint32_t Lsum_all,
                                                         uint32_t B, uint32_t stages) {
    TinySmem s;
    size_t o = 0;
    s.tabk = o;  o += B ? (size_t)Qp * 2048 : 0;
    s.tab1 = o;  o = al16(o + (size_t)Qp * A * 2);
    s.lcnt = o;  o = al16(o + 4 * (size_t)(A + 1));
    s.loff = o;  o = al16(o + 4 * (size_t)(A + 1));
    s.llist = o; o = al16(o + 4 * (size_t)Lsum_all);
    // union: TMA stage buffers during the walk, dense chunk maps afterwards
    s.uni = o = al1k(o);
    // dense maps of ONE row per lane at a time (the two rows of a lane are composed in turn),
    // rows padded (tiny_map_strides) so the per-lane row writes are bank-conflict free
    const size_t maps = al16((size_t)kT * tiny_mend_stride(Qpad)) + 4 * (size_t)kT * tiny_mhits_stride(Qpad);
    const size_t stg = (size_t)kWarps * stages * kStageBytes;
    s.mend = s.uni;
    s.mhits = s.uni + al16((size_t)kT * tiny_mend_stride(Qpad));
    o = al16(s.uni + (maps > stg ? maps : stg));
    s.wend = o;  o = al16(o + 4 * (size_t)kWarps * Qpad);
    s.whits = o; o = al16(o + 8 * (size_t)kWarps * Qpad);
    s.mbar = o;  o = al16(o + 8 * (size_t)kWarps * kMaxStages);
    s.flag = o;  o = al16(o + 16);
    s.total = o + 1024;   // slack for aligning the dynamic smem base
    return s;
}

// Register-resident routes of one chunk: e[j] is route j's current state in the table's
// address form, h[j] its hit count.
template <int K, int B>
struct Routes {
    uint32_t e[K];
    uint32_t h[K];
    uint32_t bad;

    __device__ __forceinline__ uint32_t state(int j) const { return B ? (e[j] & 0xFFFFu) >> 11 : e[j]; }

    // one symbol (any alignment), via tab1
    __device__ __forceinline__ void step1(uint32_t c, const uint16_t* __restrict__ tab1, uint32_t A, uint32_t lane4) {
        if (c >= A) {
            bad |= 0x80u;
            c = A - 1;
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint32_t t = tab1[state(j) * A + c];
            h[j] += t >> 15;
            const uint32_t s = t & 0x7FFFu;
            e[j] = B ? ((s << 11) | lane4) : s;
        }
    }

    uint32_t m16;   // the constant 16, hidden from the optimiser (PAREM_HITS_IMAD)

    __device__ __forceinline__ void group(uint32_t g7, const unsigned char* __restrict__ tabk) {
        // keep the masked group value opaque so the compiler emits ONE LOP3 per route
        // ((e & 0xFFFF) | g7) instead of folding the group mask into a second one
        asm("" : "+r"(g7));
#pragma unroll
        for (int j = 0; j < K; ++j) {
            e[j] = *reinterpret_cast<const uint32_t*>(tabk + ((e[j] & 0xFFFFu) | g7));
#ifdef PAREM_HITS_IMAD
            // h += e >> 28 on the FMA pipe (IMAD.HI with an opaque 16) -- the ALU pipe
            // carries the LOP3s
            asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(h[j]) : "r"(e[j]), "r"(m16));
#else
            h[j] += e[j] >> 28;   // LEA.HI
#endif
        }
    }

    // four symbols packed in one little-endian word
    __device__ __forceinline__ void word(uint32_t w, const unsigned char* __restrict__ tabk,
                                         const uint16_t* __restrict__ tab1, uint32_t A, uint32_t badmask,
                                         uint32_t lane4) {
        if constexpr (B == 2) {
            // (invalid bytes are flagged per 16-byte vector in vec())
            // w * 130 = w<<7 + w<<1: b0 | b1<<2 lands in bits 7..10 and b2 | b3<<2 in bits
            // 23..26; every other partial product has its own 2-bit slot (no carries).
            const uint32_t P = w * 130u;
            group(P & 0x780u, tabk);                         // symbols 0,1
            group(__umulhi(w, 0x00820000u) & 0x780u, tabk);  // symbols 2,3: (w * 130) >> 16 on the FMA pipe
        } else if constexpr (B == 1) {
            const uint32_t P = w * 0x10204080u;  // b0..b3 -> bits 28..31
            group((P >> 21) & 0x780u, tabk);
        } else {
            bad |= badbits(w, A);
            step1(w & 0xFFu, tab1, A, lane4);
            step1((w >> 8) & 0xFFu, tab1, A, lane4);
            step1((w >> 16) & 0xFFu, tab1, A, lane4);
            step1(w >> 24, tab1, A, lane4);
        }
    }

    __device__ __forceinline__ void vec(const uint4& x, const unsigned char* __restrict__ tabk,
                                        const uint16_t* __restrict__ tab1, uint32_t A, uint32_t badmask,
                                        uint32_t lane4) {
        if constexpr (B != 0) bad |= (x.x | x.y | x.z | x.w) & badmask;   // bytes >= A (C11)
        word(x.x, tabk, tab1, A, badmask, lane4);
        word(x.y, tabk, tab1, A, badmask, lane4);
        word(x.z, tabk, tab1, A, badmask, lane4);
        word(x.w, tabk, tab1, A, badmask, lane4);
    }

    // advance every route over in[a, b) read straight from global memory
    __device__ __forceinline__ void walk(const uint8_t* __restrict__ in, uint64_t a, uint64_t b,
                                         const unsigned char* __restrict__ tabk, const uint16_t* __restrict__ tab1,
                                         uint32_t A, uint32_t badmask, uint32_t lane4) {
        if (a >= b) return;
        const uint64_t mis = (uint64_t)(((uintptr_t)(in + a)) & 15u);
        uint64_t head = mis ? a + (16 - mis) : a;
        if (head > b) head = b;
        for (; a < head; ++a) step1(in[a], tab1, A, lane4);
        const uint32_t nvec = (uint32_t)((b - a) >> 4);
        const uint8_t* p = in + a;
#pragma unroll 2
        for (uint32_t v = 0; v < nvec; ++v) vec(ldg_v4(p + 16ull * v), tabk, tab1, A, badmask, lane4);
        a += (uint64_t)nvec << 4;
        for (; a < b; ++a) step1(in[a], tab1, A, lane4);
    }
};

// One chunk's A2 data: boundaries [b0, b1), candidate list R_i (Llist[loff .. loff + cnt),
// or -- look-back rule -- the set bits of `mask`), q0 for chunk 0, and |R_i| for the stats.
struct TinyChunk {
    uint64_t t, b0, b1;
    uint32_t cnt, loff, q0, rc, mask;
    bool live;
};

// j-th candidate start state of chunk c
__device__ __forceinline__ uint32_t tiny_cand(const TinyChunk& c, const uint32_t* Llist, uint32_t j) {
    return c.mask ? (uint32_t)__fns(c.mask, 0, (int)j + 1) : Llist[c.loff + j];
}

__device__ __forceinline__ TinyChunk tiny_chunk(const MatchParams& P, uint64_t t, const uint32_t* Lcnt,
                                                const uint32_t* Loff, const uint16_t* tab1) {
    TinyChunk c;
    c.t = t;
    c.live = t < P.p;
    c.b0 = c.b1 = 0;
    c.cnt = c.loff = c.q0 = c.rc = c.mask = 0;
    if (c.live && t > 0 && P.cand == PAREM_CANDIDATES_LOOKBACK) {
        // NEXT-2 (i): R = delta*(Q, T[b0 - k, b0)) n S(T[b0]) as a bit set over <= 32 states
        // (the sink of a partial table is DEAD, never a candidate: C9/C10)
        const DevDfa& d = P.d;
        c.b0 = boundary_of(P, t, Lcnt);
        c.b1 = boundary_of(P, t + 1, Lcnt);
        const uint32_t nosink = d.has_sink ? ~(1u << d.sink) : ~0u;
        uint32_t m = (d.Qp >= 32 ? ~0u : (1u << d.Qp) - 1u) & nosink;
        for (uint64_t j = c.b0 > P.lookback ? c.b0 - P.lookback : 0; j < c.b0; ++j) {
            uint32_t ch = P.in[j];
            if (ch >= d.A) ch = d.A - 1;   // ESYMBOL is reported anyway; keep the set valid
            uint32_t nm = 0;
            for (uint32_t r = m; r; r &= r - 1) nm |= 1u << (tab1[(__ffs(r) - 1) * d.A + ch] & 0x7FFFu);
            m = nm & nosink;
        }
        c.mask = m ? m : 0u;
        c.cnt = __popc(m);
        uint32_t cf = P.in[c.b0];
        if (cf >= d.A) cf = d.A - 1;
        uint32_t inS = 0;   // |R n S(c_first)|
        for (uint32_t r = m; r; r &= r - 1)
            inS += !d.has_sink || (tab1[(__ffs(r) - 1) * d.A + cf] & 0x7FFFu) != d.sink;
        c.rc = inS;
        if (!m) c.cnt = 0;
        return c;
    }
    if (c.live) {
        c.b0 = boundary_of(P, t, Lcnt);
        c.b1 = boundary_of(P, t + 1, Lcnt);
        if (t == 0 || (P.cpi && t % P.cpi == 0)) {   // first chunk (of every batch input)
            bool dead;
            c.q0 = start_state(P, &dead);
            c.cnt = 1;
            c.rc = 1;
        } else {
            const uint32_t ch = P.in[c.b0 - 1];
            const uint32_t li = (P.cand == PAREM_CANDIDATES_ENUM || ch >= P.d.A) ? P.d.A : ch;
            c.cnt = Lcnt[li];
            c.loff = Loff[li];
            c.rc = route_count(P, ch, P.in[c.b0], c.cnt);
        }
    }
    return c;
}

template <int K, int B, bool TMA>
__global__ void __launch_bounds__(kT, 1) tiny_kernel(const MatchParams P, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    // align the dynamic shared memory base to 1024 B (TMA swizzle atoms)
    unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    const DevDfa& d = P.d;
    const uint32_t Qp = d.Qp, Qpad = d.Qpad, A = d.A;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t S = TMA ? P.stages : 0u;
    const TinySmem L = tiny_layout(Qp, Qpad, A, d.Lsum_all, B, S);
    const uint32_t MS = tiny_mend_stride(Qpad), HS = tiny_mhits_stride(Qpad);
    uint32_t* tabk32 = reinterpret_cast<uint32_t*>(sm + L.tabk);
    const unsigned char* tabk = sm + L.tabk;
    uint16_t* tab1 = reinterpret_cast<uint16_t*>(sm + L.tab1);
    uint32_t* Lcnt = reinterpret_cast<uint32_t*>(sm + L.lcnt);
    uint32_t* Loff = reinterpret_cast<uint32_t*>(sm + L.loff);
    uint32_t* Llist = reinterpret_cast<uint32_t*>(sm + L.llist);
    uint8_t* mend = sm + L.mend;
    uint32_t* mhits = reinterpret_cast<uint32_t*>(sm + L.mhits);
    uint32_t* wend = reinterpret_cast<uint32_t*>(sm + L.wend);
    unsigned long long* whits = reinterpret_cast<unsigned long long*>(sm + L.whits);
    uint32_t* flag = reinterpret_cast<uint32_t*>(sm + L.flag);
    const uint32_t mbar0 = smem_u32(sm + L.mbar) + warp * kMaxStages * 8u;
    const uint32_t stage0 = smem_u32(sm + L.uni) + warp * S * kStageBytes;

    // ---- stage the tables (A1 products) into shared memory; init this warp's barriers ----
    if (B)
        for (uint32_t i = tid; i < Qp * 512u; i += kT) tabk32[i] = __ldg(d.stride + (i >> 5)) | ((i & 31u) << 2);
    for (uint32_t i = tid; i < Qp * A; i += kT) tab1[i] = __ldg(d.tab1 + i);
    for (uint32_t i = tid; i <= A; i += kT) {
        Lcnt[i] = __ldg(d.Lcnt + i);
        Loff[i] = __ldg(d.Loff + i);
    }
    for (uint32_t i = tid; i < d.Lsum_all; i += kT) Llist[i] = __ldg(d.Llist + i);
    const uint64_t row0 = (uint64_t)blockIdx.x * kRows + warp * kRowsW;   // first chunk of this warp
    const uint32_t nst = TMA ? (uint32_t)(P.L / kBoxBytes) : 0u;
    const bool warp_live = row0 < P.p;
    if (TMA && lane == 0) {
        for (uint32_t s = 0; s < S; ++s) mbar_init(mbar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the first stages do not depend on A2: start streaming before the prologue
        if (warp_live)
            for (uint32_t s = 0; s < S && s < nst; ++s) {
                mbar_expect_tx(mbar0 + 8 * s, kStageBytes);
                tma_load_2d(stage0 + s * kStageBytes, &tmap, (int32_t)(s * kBoxBytes), (int32_t)row0, mbar0 + 8 * s);
            }
    }
    __syncthreads();

    // ---- A2: this lane's two chunks (rows lane and lane + 32 of the warp's box) and R_i ----
    const TinyChunk ca = tiny_chunk(P, row0 + lane, Lcnt, Loff, tab1);
    const TinyChunk cb = tiny_chunk(P, row0 + 32 + lane, Lcnt, Loff, tab1);
    const bool act_a = ca.live && ca.cnt, act_b = cb.live && cb.cnt;
    // per-byte invalid bits for A = 1, 2, 4 (powers of two): every bit at or above log2(A)
    const uint32_t bm = B ? (0xFFu & ~(A - 1u)) * 0x01010101u : 0u;
    const uint32_t lane4 = lane << 2;

    // ---- A3 pass 0: the first K candidates of both chunks, one pass over the bytes ----
    Routes<K, B> ra, rb;
    ra.bad = rb.bad = 0;
    ra.m16 = 16;
    asm volatile("" : "+r"(ra.m16));
    rb.m16 = ra.m16;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const uint32_t ka = ca.cnt ? min((uint32_t)j, ca.cnt - 1) : 0;
        const uint32_t kb = cb.cnt ? min((uint32_t)j, cb.cnt - 1) : 0;
        const bool sta = ca.t == 0 || (P.cpi && ca.t % P.cpi == 0), stb = P.cpi && cb.t % P.cpi == 0;
        const uint32_t sa = sta ? ca.q0 : (ca.cnt ? tiny_cand(ca, Llist, ka) : 0u);
        const uint32_t sb = stb ? cb.q0 : (cb.cnt ? tiny_cand(cb, Llist, kb) : 0u);
        ra.e[j] = B ? ((sa << 11) | lane4) : sa;
        rb.e[j] = B ? ((sb << 11) | lane4) : sb;
        ra.h[j] = rb.h[j] = 0;
    }
    if (TMA) {
        const uint64_t xa0 = ca.t * P.L, xb0 = cb.t * P.L;   // nominal row starts
        // first staged byte each chunk uses (units before it belong to the scalar head)
        const uint32_t srel_a = act_a ? (uint32_t)((ca.b0 - xa0 + 15) & ~15ull) : 0xFFFFFFFFu;
        const uint32_t srel_b = act_b ? (uint32_t)((cb.b0 - xb0 + 15) & ~15ull) : 0xFFFFFFFFu;
        if (act_a) ra.walk(P.in, ca.b0, min(xa0 + srel_a, ca.b1), tabk, tab1, A, bm, lane4);
        if (act_b) rb.walk(P.in, cb.b0, min(xb0 + srel_b, cb.b1), tabk, tab1, A, bm, lane4);
        if (warp_live) {
            // SWIZZLE_64B: 16-byte unit u of row l sits at unit u ^ ((l >> 1) & 3); rows l and
            // l + 32 share the pattern
            const uint32_t sw = (lane >> 1) & 3u, offa = lane * kBoxBytes, offb = (lane + 32u) * kBoxBytes;
            auto next_stage = [&](uint32_t s, uint32_t slot) {
                __syncwarp();
                if (lane == 0 && s + S < nst) {
                    mbar_expect_tx(mbar0 + 8 * slot, kStageBytes);
                    tma_load_2d(stage0 + slot * kStageBytes, &tmap, (int32_t)((s + S) * kBoxBytes), (int32_t)row0,
                                mbar0 + 8 * slot);
                }
            };
            // advance both chunks' routes over stage s.  Only stages 0 and 1 can hold head
            // units (SNAP moves a boundary <= 64 bytes), so later stages run unguarded: an
            // inactive chunk walks harmless garbage (zero-filled rows past p) and is discarded.
            auto run_stage = [&](auto& xa, auto& xb, uint32_t s, uint32_t buf) {
                if (s < 2) {
                    const uint32_t rel = s * kBoxBytes;
#pragma unroll 1
                    for (uint32_t u = 0; u < 4; ++u) {
                        const uint32_t ou = (u ^ sw) << 4;
                        if (rel + 16 * u >= srel_a) xa.vec(lds128(buf + offa + ou), tabk, tab1, A, bm, lane4);
                        if (rel + 16 * u >= srel_b) xb.vec(lds128(buf + offb + ou), tabk, tab1, A, bm, lane4);
                    }
                } else {
#pragma unroll
                    for (uint32_t u = 0; u < 4; ++u) {
                        const uint32_t ou = (u ^ sw) << 4;
                        const uint4 va = lds128(buf + offa + ou);
                        const uint4 vb = lds128(buf + offb + ou);
                        xa.vec(va, tabk, tab1, A, bm, lane4);
                        xb.vec(vb, tabk, tab1, A, bm, lane4);
                    }
                }
            };
            uint32_t s = 0, slot = 0, phase = 0;
            auto advance = [&]() {
                if (++slot == S) {
                    slot = 0;
                    phase ^= 1u;
                }
                ++s;
            };
            if constexpr (K > 1) {
                // Route merging: routes of one chunk that reach the same state stay together
                // for the rest of the chunk.  Once EVERY lane of the warp has all K routes of
                // both its chunks in one state (checked per stage, warp-uniform), the warp
                // advances a single route per chunk and rebuilds the others exactly: end =
                // shared end, hits = shared hits + the per-route offset at the merge point.
                while (s < nst) {
                    mbar_wait(mbar0 + 8 * slot, phase);
                    run_stage(ra, rb, s, stage0 + slot * kStageBytes);
                    next_stage(s, slot);
                    advance();
                    bool conv = true;
#pragma unroll
                    for (int j = 1; j < K; ++j) conv &= (ra.e[j] == ra.e[0] || !act_a) && (rb.e[j] == rb.e[0] || !act_b);
                    if (__all_sync(0xFFFFFFFFu, conv)) break;
                }
                if (s < nst) {
                    Routes<1, B> qa, qb;
                    qa.e[0] = ra.e[0];
                    qa.h[0] = ra.h[0];
                    qb.e[0] = rb.e[0];
                    qb.h[0] = rb.h[0];
                    qa.bad = qb.bad = 0;
                    qa.m16 = qb.m16 = ra.m16;
                    while (s < nst) {
                        mbar_wait(mbar0 + 8 * slot, phase);
                        run_stage(qa, qb, s, stage0 + slot * kStageBytes);
                        next_stage(s, slot);
                        advance();
                    }
                    const uint32_t ha = ra.h[0], hb = rb.h[0];
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        ra.h[j] = qa.h[0] + (ra.h[j] - ha);   // u32 wrap-around is exact here
                        ra.e[j] = qa.e[0];
                        rb.h[j] = qb.h[0] + (rb.h[j] - hb);
                        rb.e[j] = qb.e[0];
                    }
                    ra.bad |= qa.bad;
                    rb.bad |= qb.bad;
                }
            } else {
                while (s < nst) {
                    mbar_wait(mbar0 + 8 * slot, phase);
                    run_stage(ra, rb, s, stage0 + slot * kStageBytes);
                    next_stage(s, slot);
                    advance();
                }
            }
        }
        if (act_a) ra.walk(P.in, xa0 + P.L, ca.b1, tabk, tab1, A, bm, lane4);   // tails past the rows
        if (act_b) rb.walk(P.in, xb0 + P.L, cb.b1, tabk, tab1, A, bm, lane4);
    } else {
        if (act_a) ra.walk(P.in, ca.b0, ca.b1, tabk, tab1, A, bm, lane4);
        if (act_b) rb.walk(P.in, cb.b0, cb.b1, tabk, tab1, A, bm, lane4);
    }
    __syncthreads();   // stage buffers are dead from here on: they become the chunk maps

    // ---- per-chunk dense maps (identity for non-candidates), extra passes, validation ----
    auto finish = [&](const TinyChunk& c, Routes<K, B>& r, bool act, uint32_t lr) {
        for (uint32_t q = 0; q < Qpad; ++q) {
            mend[lr * MS + q] = (uint8_t)q;
            mhits[lr * HS + q] = 0;
        }
        if (!c.live) return;
        uint32_t badacc = act ? r.bad : 0u;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((uint32_t)j < c.cnt) {
                const uint32_t s = (c.t == 0 || (P.cpi && c.t % P.cpi == 0)) ? c.q0 : tiny_cand(c, Llist, j);
                mend[lr * MS + s] = (uint8_t)r.state(j);
                mhits[lr * HS + s] = r.h[j];
            }
        // extra passes for chunks with more than K candidates (SNAP window miss, Enum)
        for (uint32_t base = K; base < c.cnt; base += K) {
            Routes<K, B> x;
            x.bad = 0;
            x.m16 = r.m16;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const uint32_t s = tiny_cand(c, Llist, min(base + (uint32_t)j, c.cnt - 1));
                x.e[j] = B ? ((s << 11) | lane4) : s;
                x.h[j] = 0;
            }
            x.walk(P.in, c.b0, c.b1, tabk, tab1, A, bm, lane4);
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (base + (uint32_t)j < c.cnt) {
                    const uint32_t s = tiny_cand(c, Llist, base + j);
                    mend[lr * MS + s] = (uint8_t)x.state(j);
                    mhits[lr * HS + s] = x.h[j];
                }
        }
        if (P.fmend) {   // parem_find_async: keep this chunk's dense map for the position pass
            for (uint32_t q = 0; q < Qpad; ++q) {
                P.fmend[c.t * Qpad + q] = mend[lr * MS + q];
                P.fmhits[c.t * Qpad + q] = mhits[lr * HS + q];
            }
        }
        if (c.cnt == 0 && first_bad(P.in, c.b0, c.b1, A) < c.b1) badacc = 1;   // R_i empty: still validate
        if (badacc) {
            const uint64_t off = first_bad(P.in, c.b0, c.b1, A);
            if (off < c.b1) {
                if (P.cpi) atomicMax(P.bstats + 4 * (c.t / P.cpi), ~(unsigned long long)(off - (c.t / P.cpi) * P.n_one));
                else atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
            }
        }
    };
    // ---- A4 (first level): each warp composes its 64 chunk maps in row order, lane q =
    // start state q: rows lane (chunk a) first, then rows 32 + lane (chunk b) ----
    uint32_t wce = lane < Qpad ? lane : 0;
    unsigned long long wch = 0;
    auto compose32 = [&]() {
        __syncwarp();
        for (uint32_t i = 0; i < 32; ++i) {
            const uint32_t r = warp * 32 + i;
            const uint32_t ne = mend[r * MS + wce];
            wch += mhits[r * HS + wce];
            wce = ne;
        }
        __syncwarp();
    };
    finish(ca, ra, act_a, warp * 32 + lane);
    compose32();
    finish(cb, rb, act_b, warp * 32 + lane);
    compose32();
    if (lane < Qpad) {
        wend[warp * Qpad + lane] = wce;
        whits[warp * Qpad + lane] = wch;
    }

    // ---- stats (warp reduce -> atomics) ----
    {
        const uint32_t rs = warp_sum(ca.rc + cb.rc);
        const unsigned long long ss = warp_sum((ca.live ? (unsigned long long)ca.rc * (ca.b1 - ca.b0) : 0ull) +
                                               (cb.live ? (unsigned long long)cb.rc * (cb.b1 - cb.b0) : 0ull));
        if (lane == 0 && rs) {
            // a warp's 64 chunks never span two batch inputs (inputs are whole numbers of warps)
            unsigned long long* st = P.cpi ? P.bstats + 4 * (row0 / P.cpi) + 1 : &P.hdr->routes;
            atomicAdd(st, (unsigned long long)rs);
            atomicAdd(st + 1, ss);
        }
    }
    __syncthreads();

    // Tile maps.  A batch of SHORT inputs (cpi < kRows chunks each, a whole number of warps)
    // packs spt = kRows / cpi inputs into one CTA tile: warp j composes the warp maps of
    // sub-tile j only, so no map ever spans two inputs and chunks can stay long.
    unsigned long long* tiles = reinterpret_cast<unsigned long long*>(P.maps);
    const uint32_t spt = (P.cpi && P.cpi < kRows) ? kRows / (uint32_t)P.cpi : 1u;
    if (warp < spt) {
        const uint32_t wps = kWarps / spt;
        uint32_t ce = lane < Qpad ? lane : 0;
        unsigned long long ch = 0;
        for (uint32_t w = warp * wps; w < (warp + 1) * wps; ++w) {
            const uint32_t row = w * Qpad + ce;
            const uint32_t ne = wend[row];
            ch += whits[row];
            ce = ne;
        }
        if (lane < Qpad) tiles[((uint64_t)blockIdx.x * spt + warp) * Qpad + lane] = (ch << 8) | ce;
        __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&P.hdr->done, 1u);
        *flag = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!*flag) return;
    __threadfence();

    if (P.cpi) {   // batch: one fold per input, warp w takes inputs w, w + 16, ...
        const uint32_t tpi = P.cpi >= kRows ? (uint32_t)(P.cpi / kRows) : 1u;   // maps per input
        const uint32_t nin = (uint32_t)(P.p / P.cpi);
        for (uint32_t b = warp; b < nin; b += kWarps) {
            uint32_t ce = lane < Qpad ? lane : 0;
            unsigned long long ch = 0;
            for (uint32_t i = 0; i < tpi; ++i) {
                const unsigned long long m =
                    lane < Qpad ? ld_cg_u64(tiles + (uint64_t)(b * tpi + i) * Qpad + lane) : (unsigned long long)lane;
                const uint32_t ne = __shfl_sync(0xFFFFFFFFu, (uint32_t)(m & 0xFFu), ce);
                const unsigned long long nh = __shfl_sync(0xFFFFFFFFu, m >> 8, ce);
                ch += nh;
                ce = ne;
            }
            bool dead;
            const uint32_t q0 = start_state(P, &dead);
            const uint32_t qf = __shfl_sync(0xFFFFFFFFu, ce, q0);
            const unsigned long long hf = __shfl_sync(0xFFFFFFFFu, ch, q0);
            if (lane == 0) {
                unsigned long long* st = P.bstats + 4 * b;
                const bool sdead = P.d.has_sink && qf == P.d.sink;
                parem_result r;
                r.final_state = sdead ? PAREM_DEAD : qf;
                r.accepted = sdead ? 0u : (uint32_t)P.d.acc[qf];
                r.match_count = hf;
                r.num_chunks = P.cpi;
                r.routes = st[1];
                r.route_steps = st[2];
                r.lookups_k = 0;
                r.status = st[0] ? PAREM_ESYMBOL : PAREM_OK;
                r.bad_offset = st[0] ? ~st[0] : 0ull;
                P.results[b] = r;
                st[0] = st[1] = st[2] = 0ull;   // leave the workspace clean (PAREM_FLAG_WS_CLEAN)
            }
        }
        __syncthreads();
        if (tid == 0) reset_header(P);
        return;
    }
    // ---- last CTA: fold the tile maps along q0's path (lane q = start q, shuffles) ----
    const uint32_t G = gridDim.x;
    const uint32_t per = (G + kWarps - 1) / kWarps;
    const uint32_t lo = min(G, warp * per), hi = min(G, lo + per);
    uint32_t ce = lane < Qpad ? lane : 0;
    unsigned long long ch = 0;
    for (uint32_t i0 = lo; i0 < hi; i0 += 8) {   // 8 tile maps loaded at once, then chained
        unsigned long long m[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            m[j] = (i0 + j < hi && lane < Qpad) ? ld_cg_u64(tiles + (uint64_t)(i0 + j) * Qpad + lane)
                                               : (unsigned long long)lane;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            const uint32_t ne = __shfl_sync(0xFFFFFFFFu, (uint32_t)(m[j] & 0xFFu), ce);
            const unsigned long long nh = __shfl_sync(0xFFFFFFFFu, m[j] >> 8, ce);
            if (i0 + j < hi) {
                ch += nh;
                ce = ne;
            }
        }
    }
    if (lane < Qpad) {
        wend[warp * Qpad + lane] = ce;
        whits[warp * Qpad + lane] = ch;
    }
    __syncthreads();
    if (tid == 0) {
        bool dead;
        uint32_t q = start_state(P, &dead);
        unsigned long long hits = 0;
        for (uint32_t w = 0; w < kWarps; ++w) {
            hits += whits[w * Qpad + q];
            q = wend[w * Qpad + q];
        }
        write_result(P, q, hits, dead);
    }
}

template <int K, int B, bool TMA>
const void* tiny_fn() {
    return reinterpret_cast<const void*>(&tiny_kernel<K, B, TMA>);
}

}  // namespace
}  // namespace parem
