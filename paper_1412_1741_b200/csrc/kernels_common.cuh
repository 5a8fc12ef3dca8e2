// kernels_common.cuh -- device helpers shared by the tiny and lanes kernels:
// chunk boundaries (Alg. 1 lines 3-4, with the planner's SNAP policy),
// the candidate set R_i, byte validation (reading C11) and the
// result epilogue (P:58 acceptance, P:70 join on q0's path).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace parem {

__device__ __forceinline__ uint4 ldg_v4(const uint8_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// streaming input: do not allocate in L1 (keeps L1 for L2-resident transition tables)
__device__ __forceinline__ uint4 ldg_v4_na(const uint8_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned long long ld_cg_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Per-byte validity (reading C11): returns a word whose bit 7 of byte k is set iff byte k of
// w is >= A.  Exact for every A in [1, 256].
__device__ __forceinline__ uint32_t badbits(uint32_t w, uint32_t A) {
    if (A >= 256) return 0u;
    if (A <= 128) {
        // (b | 0x80) - A has bit 7 clear iff b < A (for b < 128); b >= 128 is caught by "| w"
        return (((w | 0x80808080u) - A * 0x01010101u) | w) & 0x80808080u;
    }
    // A in 129..255: bad iff b >= 128 and (b & 0x7f) >= A - 128
    return (((w & 0x7F7F7F7Fu) | 0x80808080u) - (A - 128u) * 0x01010101u) & w & 0x80808080u;
}

// Boundary b_i of chunk i (0 <= i <= p).  GRID: b_i = i * L, b_p = n (remainder to the last
// chunk, reading C7).  SNAP: the planner moves b_i forward within [x, min(x + win, n - 1)],
// x = i * L, to the first position minimising |L(T[b - 1])| (ties: smallest b) -- the
// paper's rule R = S n L is then applied at the moved boundary.  Both neighbouring chunks
// evaluate the same deterministic function, so the partition is consistent.
__device__ __forceinline__ uint64_t boundary_of(const MatchParams& P, uint64_t i, const uint32_t* Lcnt) {
    if (i == 0) return 0;
    if (i >= P.p) return P.n;
    const uint64_t x = i * P.L;
    if (P.policy != PAREM_BOUNDARY_SNAP || P.win == 0) return x;
    uint64_t hi = x + P.win;
    if (hi > P.n - 1) hi = P.n - 1;
    uint32_t best = 0xFFFFFFFFu;
    uint64_t by = x;
    for (uint64_t y = x; y <= hi; ++y) {
        const uint32_t c = __ldg(P.in + y - 1);
        const uint32_t k = c < P.d.A ? Lcnt[c] : 0xFFFFFFFEu;
        if (k < best) {
            best = k;
            by = y;
            if (k <= P.d.Lmin) break;
        }
    }
    return by;
}

// Start state of chunk 0 ("already knows the possible initial state, q0"), or the
// carried state of a previous segment (parem_match_continue_async).
__device__ __forceinline__ uint32_t start_state(const MatchParams& P, bool* dead) {
    *dead = false;
    if (P.carry) {
        const uint32_t s = P.carry->final_state;
        if (s == PAREM_DEAD || s >= P.d.Q) {
            *dead = true;
            return 0;
        }
        return s;
    }
    return P.d.start;
}

// |R_i| for the stats: |L(c_last) n S(c_first)|; = |L(c_last)| for complete tables.
__device__ __forceinline__ uint32_t route_count(const MatchParams& P, uint32_t c_last, uint32_t c_first,
                                                uint32_t cnt) {
    if (P.cand == PAREM_CANDIDATES_ENUM) return P.d.Q;
    if (P.d.Rcnt && c_last < P.d.A && c_first < P.d.A) return __ldg(P.d.Rcnt + c_last * P.d.A + c_first);
    return cnt;
}

// First offset in [a, b) holding a byte >= A (slow path, only after a detection).
__device__ __forceinline__ uint64_t first_bad(const uint8_t* in, uint64_t a, uint64_t b, uint32_t A) {
    if (A >= 256u) return b;   // every byte is a symbol
    uint64_t k = a;
    for (; k < b && (((uintptr_t)(in + k)) & 15u); ++k)
        if (in[k] >= A) return k;
    // 16 bytes at a time: byte x >= A iff x + (256 - A) carries out of bit 7
    const uint32_t K = (256u - A) * 0x01010101u, K7 = K & 0x7F7F7F7Fu;
    for (; k + 16 <= b; k += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(in + k));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t bad = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) bad |= (w[q] & K) | ((w[q] | K) & ((w[q] & 0x7F7F7F7Fu) + K7));
        if (bad & 0x80808080u) break;   // the byte loop below finds the offset
    }
    for (; k < b; ++k)
        if (in[k] >= A) return k;
    return b;
}

// Every completed match leaves its workspace header zeroed (PAREM_FLAG_WS_CLEAN): the
// last CTA calls this after reading the header.
__device__ __forceinline__ void reset_header(const MatchParams& P) {
    volatile WsHeader* h = P.hdr;
    h->done = 0;
    h->err = 0;
    h->bad_inv = 0;
    h->routes = 0;
    h->steps = 0;
    h->hits = 0;
    h->lookups = 0;
    h->final_q = 0;
    __threadfence();
}

// Epilogue, run by one thread of the last CTA: q is the internal state reached from the
// start state, hits the matches counted on that path (u64).
__device__ __forceinline__ void write_result(const MatchParams& P, uint32_t q, unsigned long long hits,
                                             bool start_dead) {
    uint64_t base_count = 0, base_chunks = 0, base_routes = 0, base_steps = 0, cbad = 0;
    int32_t cst = PAREM_OK;
    if (P.carry) {
        const volatile parem_result* c = P.carry;
        base_count = c->match_count;
        base_chunks = c->num_chunks;
        base_routes = c->routes;
        base_steps = c->route_steps;
        cst = c->status;
        cbad = c->bad_offset;
    }
    volatile WsHeader* h = P.hdr;
    const bool dead = start_dead || (P.d.has_sink && q == P.d.sink);
    parem_result r;
    r.final_state = dead ? PAREM_DEAD : q;
    r.accepted = dead ? 0u : (uint32_t)P.d.acc[q];
    r.match_count = base_count + (start_dead ? 0ull : hits);
    r.num_chunks = base_chunks + P.p;
    r.routes = base_routes + h->routes;
    r.route_steps = base_steps + h->steps;
    r.lookups_k = (uint32_t)min((h->lookups + 1023ull) >> 10, 0xFFFFFFFFull);
    const unsigned long long binv = h->bad_inv;
    if (cst == PAREM_ESYMBOL) {
        r.status = cst;
        r.bad_offset = cbad;
    } else if (binv != 0ull) {
        r.status = PAREM_ESYMBOL;
        r.bad_offset = P.offset_base + ~binv;
    } else {
        r.status = cst;
        r.bad_offset = 0;
    }
    *P.result = r;
    reset_header(P);
}

// ---- TMA / mbarrier helpers (tiny kernel, converging follow walk) ----
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

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

}  // namespace parem
