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

constexpr uint32_t kT = kTinyThreads;       // 512 threads = 512 chunks per CTA
constexpr uint32_t kWarps = kT / 32;
constexpr uint32_t kBoxBytes = 64;          // TMA box: 32 rows x 64 bytes
constexpr uint32_t kStageBytes = 32 * kBoxBytes;
constexpr uint32_t kStages = 2;

__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ __forceinline__ size_t al1k(size_t x) { return (x + 1023) & ~(size_t)1023; }

struct TinySmem {
    size_t tabk, tab1, lcnt, loff, llist, uni, mend, mhits, wend, whits, mbar, flag, total;
};

// Offsets relative to a 1024-aligned base (the kernel aligns the dynamic smem pointer).
__host__ __device__ __forceinline__ TinySmem tiny_layout(uint32_t Qp, uint32_t Qpad, uint32_t A, uint32_t Lsum_all,
                                                         uint32_t B, bool tma) {
    TinySmem s;
    size_t o = 0;
    s.tabk = o;  o += B ? (size_t)Qp * 2048 : 0;
    s.tab1 = o;  o = al16(o + (size_t)Qp * A * 2);
    s.lcnt = o;  o = al16(o + 4 * (size_t)(A + 1));
    s.loff = o;  o = al16(o + 4 * (size_t)(A + 1));
    s.llist = o; o = al16(o + 4 * (size_t)Lsum_all);
    // union: TMA stage buffers during the walk, dense chunk maps afterwards
    s.uni = o = al1k(o);
    const size_t maps = al16((size_t)kT * Qpad) + 4 * (size_t)kT * Qpad;
    const size_t stages = tma ? (size_t)kWarps * kStages * kStageBytes : 0;
    s.mend = s.uni;
    s.mhits = s.uni + al16((size_t)kT * Qpad);
    o = al16(s.uni + (maps > stages ? maps : stages));
    s.wend = o;  o = al16(o + 4 * (size_t)kWarps * Qpad);
    s.whits = o; o = al16(o + 8 * (size_t)kWarps * Qpad);
    s.mbar = o;  o = al16(o + 8 * (size_t)kWarps * kStages);
    s.flag = o;  o = al16(o + 16);
    s.total = o + 1024;   // slack for aligning the dynamic smem base
    return s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    // bounded spin: a lost transaction traps instead of hanging the GPU
    for (uint32_t i = 0; !mbar_try_wait(a, parity); ++i)
        if (i > (1u << 26)) __trap();
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
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
            bad |= w & badmask;
            // w * 130 = w<<7 + w<<1: b0 | b1<<2 lands in bits 7..10 and b2 | b3<<2 in bits
            // 23..26; every other partial product has its own 2-bit slot (no carries).
            const uint32_t P = w * 130u;
            group(P & 0x780u, tabk);                         // symbols 0,1
            group(__umulhi(w, 0x00820000u) & 0x780u, tabk);  // symbols 2,3: (w * 130) >> 16 on the FMA pipe
        } else if constexpr (B == 1) {
            bad |= w & badmask;
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

template <int K, int B, bool TMA>
__global__ void __launch_bounds__(kT) tiny_kernel(const MatchParams P, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    // align the dynamic shared memory base to 1024 B (TMA swizzle atoms)
    unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    const DevDfa& d = P.d;
    const uint32_t Qp = d.Qp, Qpad = d.Qpad, A = d.A;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const TinySmem L = tiny_layout(Qp, Qpad, A, d.Lsum_all, B, TMA);
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
    const uint32_t mbar0 = smem_u32(sm + L.mbar) + warp * kStages * 8u;
    const uint32_t stage0 = smem_u32(sm + L.uni) + warp * kStages * kStageBytes;

    // ---- stage the tables (A1 products) into shared memory; init this warp's barriers ----
    if (B)
        for (uint32_t i = tid; i < Qp * 512u; i += kT) tabk32[i] = __ldg(d.stride + (i >> 5)) | ((i & 31u) << 2);
    for (uint32_t i = tid; i < Qp * A; i += kT) tab1[i] = __ldg(d.tab1 + i);
    for (uint32_t i = tid; i <= A; i += kT) {
        Lcnt[i] = __ldg(d.Lcnt + i);
        Loff[i] = __ldg(d.Loff + i);
    }
    for (uint32_t i = tid; i < d.Lsum_all; i += kT) Llist[i] = __ldg(d.Llist + i);
    if (TMA && lane == 0) {
        for (uint32_t s = 0; s < kStages; ++s) mbar_init(mbar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // ---- A2: this thread's chunk and its candidate set R_i ----
    const uint64_t row0 = (uint64_t)blockIdx.x * kT + warp * 32u;   // first chunk of this warp
    const uint64_t t = row0 + lane;
    const bool live = t < P.p;
    uint64_t b0 = 0, b1 = 0;
    uint32_t cnt = 0, loff = 0, q0 = 0, rc = 0;
    if (live) {
        b0 = boundary_of(P, t, Lcnt);
        b1 = boundary_of(P, t + 1, Lcnt);
        if (t == 0) {
            bool dead;
            q0 = start_state(P, &dead);
            cnt = 1;
            rc = 1;
        } else {
            const uint32_t c = P.in[b0 - 1];
            const uint32_t li = (P.cand == PAREM_CANDIDATES_ENUM || c >= A) ? A : c;
            cnt = Lcnt[li];
            loff = Loff[li];
            rc = route_count(P, c, P.in[b0], cnt);
        }
    }
    // per-byte invalid bits for A = 1, 2, 4 (powers of two): every bit at or above log2(A)
    const uint32_t bm = B ? (0xFFu & ~(A - 1u)) * 0x01010101u : 0u;
    const uint32_t lane4 = lane << 2;
    uint32_t badacc = 0;

    // ---- A3 pass 0: the first K candidates, one pass over the chunk ----
    Routes<K, B> r;
    r.bad = 0;
    r.m16 = 16;
    asm volatile("" : "+r"(r.m16));
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const uint32_t k = cnt ? min((uint32_t)j, cnt - 1) : 0;
        const uint32_t s = t == 0 ? q0 : (cnt ? Llist[loff + k] : 0u);
        r.e[j] = B ? ((s << 11) | lane4) : s;
        r.h[j] = 0;
    }
    if (TMA) {
        // rows [row0, row0 + 32) of the tensor view; every lane walks its own row
        const uint32_t nst = (uint32_t)(P.L / kBoxBytes);
        const bool warp_live = row0 < P.p;
        const uint64_t x0 = t * P.L;                       // nominal start of the row
        const uint32_t srel = live ? (uint32_t)((b0 - x0 + 15) & ~15ull) : 0xFFFFFFFFu;  // first staged byte used
        if (live && cnt) r.walk(P.in, b0, min(x0 + srel, b1), tabk, tab1, A, bm, lane4);   // unaligned head
        if (warp_live) {
            if (lane == 0)
                for (uint32_t s = 0; s < kStages && s < nst; ++s) {
                    mbar_expect_tx(mbar0 + 8 * s, kStageBytes);
                    tma_load_2d(stage0 + s * kStageBytes, &tmap, (int32_t)(s * kBoxBytes), (int32_t)row0, mbar0 + 8 * s);
                }
            // this lane's four 16-byte units of its 64-byte row in a stage (SWIZZLE_64B:
            // unit u of row l sits at unit u ^ ((l >> 1) & 3))
            const uint32_t sw = (lane >> 1) & 3u, rowoff = lane * kBoxBytes;
            const uint32_t o0 = rowoff + ((0u ^ sw) << 4), o1 = rowoff + ((1u ^ sw) << 4),
                           o2 = rowoff + ((2u ^ sw) << 4), o3 = rowoff + ((3u ^ sw) << 4);
            const bool act = live && cnt;
            auto next_stage = [&](uint32_t s, uint32_t slot) {
                __syncwarp();
                if (lane == 0 && s + kStages < nst) {
                    mbar_expect_tx(mbar0 + 8 * slot, kStageBytes);
                    tma_load_2d(stage0 + slot * kStageBytes, &tmap, (int32_t)((s + kStages) * kBoxBytes),
                                (int32_t)row0, mbar0 + 8 * slot);
                }
            };
            // advance routes `x` over stage s (units before srel belong to the scalar head;
            // only stages 0 and 1 can hold such units, so later stages are unguarded)
            auto run_stage = [&](auto& x, uint32_t s, uint32_t buf) {
                if (!act) return;
                if (s < 2) {
                    const uint32_t rel = s * kBoxBytes;
                    if (rel + 0 >= srel) x.vec(lds128(buf + o0), tabk, tab1, A, bm, lane4);
                    if (rel + 16 >= srel) x.vec(lds128(buf + o1), tabk, tab1, A, bm, lane4);
                    if (rel + 32 >= srel) x.vec(lds128(buf + o2), tabk, tab1, A, bm, lane4);
                    if (rel + 48 >= srel) x.vec(lds128(buf + o3), tabk, tab1, A, bm, lane4);
                } else {
                    x.vec(lds128(buf + o0), tabk, tab1, A, bm, lane4);
                    x.vec(lds128(buf + o1), tabk, tab1, A, bm, lane4);
                    x.vec(lds128(buf + o2), tabk, tab1, A, bm, lane4);
                    x.vec(lds128(buf + o3), tabk, tab1, A, bm, lane4);
                }
            };
            uint32_t s = 0;
            if constexpr (K > 1) {
                // Route merging: routes of one chunk that reach the same state stay together
                // for the rest of the chunk.  Once EVERY lane of the warp has all K routes in
                // one state (checked per stage, warp-uniform), the warp advances a single
                // route and rebuilds the others exactly: end = shared end, hits = shared hits
                // + the per-route offset at the merge point.  Results are unchanged.
                for (; s < nst; ++s) {
                    const uint32_t slot = s % kStages;
                    mbar_wait(mbar0 + 8 * slot, (s / kStages) & 1u);
                    run_stage(r, s, stage0 + slot * kStageBytes);
                    next_stage(s, slot);
                    bool conv = true;
#pragma unroll
                    for (int j = 1; j < K; ++j) conv &= r.e[j] == r.e[0];
                    if (__all_sync(0xFFFFFFFFu, conv || !act)) {
                        ++s;
                        break;
                    }
                }
                if (s < nst) {
                    Routes<1, B> r1;
                    r1.e[0] = r.e[0];
                    r1.h[0] = r.h[0];
                    r1.bad = 0;
                    r1.m16 = r.m16;
                    for (; s < nst; ++s) {
                        const uint32_t slot = s % kStages;
                        mbar_wait(mbar0 + 8 * slot, (s / kStages) & 1u);
                        run_stage(r1, s, stage0 + slot * kStageBytes);
                        next_stage(s, slot);
                    }
                    const uint32_t h0 = r.h[0];
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        r.h[j] = r1.h[0] + (r.h[j] - h0);   // u32 wrap-around is exact here
                        r.e[j] = r1.e[0];
                    }
                    r.bad |= r1.bad;
                }
            } else {
                for (; s < nst; ++s) {
                    const uint32_t slot = s % kStages;
                    mbar_wait(mbar0 + 8 * slot, (s / kStages) & 1u);
                    run_stage(r, s, stage0 + slot * kStageBytes);
                    next_stage(s, slot);
                }
            }
        }
        if (live && cnt) r.walk(P.in, x0 + P.L, b1, tabk, tab1, A, bm, lane4);   // tail past the row
    } else if (live && cnt) {
        r.walk(P.in, b0, b1, tabk, tab1, A, bm, lane4);
    }
    badacc |= r.bad;
    __syncthreads();   // stage buffers are dead from here on: they become the chunk maps

    for (uint32_t q = 0; q < Qpad; ++q) {      // identity map: non-candidates keep their state
        mend[tid * Qpad + q] = (uint8_t)q;
        mhits[tid * Qpad + q] = 0;
    }
    if (live) {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((uint32_t)j < cnt) {
                const uint32_t s = t == 0 ? q0 : Llist[loff + j];
                mend[tid * Qpad + s] = (uint8_t)r.state(j);
                mhits[tid * Qpad + s] = r.h[j];
            }
        // extra passes for chunks with more than K candidates (SNAP window miss, Enum)
        for (uint32_t base = K; base < cnt; base += K) {
            Routes<K, B> x;
            x.bad = 0;
            x.m16 = r.m16;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const uint32_t s = Llist[loff + min(base + (uint32_t)j, cnt - 1)];
                x.e[j] = B ? ((s << 11) | lane4) : s;
                x.h[j] = 0;
            }
            x.walk(P.in, b0, b1, tabk, tab1, A, bm, lane4);
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (base + (uint32_t)j < cnt) {
                    const uint32_t s = Llist[loff + base + j];
                    mend[tid * Qpad + s] = (uint8_t)x.state(j);
                    mhits[tid * Qpad + s] = x.h[j];
                }
        }
        if (cnt == 0 && first_bad(P.in, b0, b1, A) < b1) badacc = 1;   // R_i empty: still validate
        if (badacc) {
            const uint64_t off = first_bad(P.in, b0, b1, A);
            if (off < b1) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
        }
    }

    // ---- stats (warp reduce -> atomics) ----
    {
        const uint32_t rs = warp_sum(rc);
        const unsigned long long ss = warp_sum(live ? (unsigned long long)rc * (b1 - b0) : 0ull);
        if (lane == 0 && rs) {
            atomicAdd(&P.hdr->routes, (unsigned long long)rs);
            atomicAdd(&P.hdr->steps, ss);
        }
    }
    __syncthreads();

    // ---- A4: compose the 32 chunk maps of each warp (lane q = start state q) ----
    {
        uint32_t ce = lane < Qpad ? lane : 0;
        unsigned long long ch = 0;
        for (uint32_t i = 0; i < 32; ++i) {
            const uint32_t row = (warp * 32 + i) * Qpad + ce;
            const uint32_t ne = mend[row];
            ch += mhits[row];
            ce = ne;
        }
        if (lane < Qpad) {
            wend[warp * Qpad + lane] = ce;
            whits[warp * Qpad + lane] = ch;
        }
    }
    __syncthreads();
    unsigned long long* tiles = reinterpret_cast<unsigned long long*>(P.maps);
    if (warp == 0) {
        uint32_t ce = lane < Qpad ? lane : 0;
        unsigned long long ch = 0;
        for (uint32_t w = 0; w < kWarps; ++w) {
            const uint32_t row = w * Qpad + ce;
            const uint32_t ne = wend[row];
            ch += whits[row];
            ce = ne;
        }
        if (lane < Qpad) tiles[(uint64_t)blockIdx.x * Qpad + lane] = (ch << 8) | ce;
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

    // ---- last CTA: fold the tile maps along q0's path (lane q = start q, shuffles) ----
    const uint32_t G = gridDim.x;
    const uint32_t per = (G + kWarps - 1) / kWarps;
    const uint32_t lo = min(G, warp * per), hi = min(G, lo + per);
    uint32_t ce = lane < Qpad ? lane : 0;
    unsigned long long ch = 0;
    for (uint32_t i = lo; i < hi; ++i) {
        const unsigned long long m = lane < Qpad ? ld_cg_u64(tiles + (uint64_t)i * Qpad + lane) : (unsigned long long)lane;
        const uint32_t ne = __shfl_sync(0xFFFFFFFFu, (uint32_t)(m & 0xFFu), ce);
        const unsigned long long nh = __shfl_sync(0xFFFFFFFFu, m >> 8, ce);
        ch += nh;
        ce = ne;
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
