// kernels_lanes.cu -- multi-start chunk simulation for large DFAs (internal states > 32):
// a GROUP of warps per chunk (several chunks per CTA share one staged table), the chunk's
// candidate start states R_i spread over the group's lanes (U per thread for ILP), all
// lanes consuming the SAME byte each step (broadcast 16-byte loads), so step k's lookups
// all hit column T[k] of the symbol-major table -- shared memory when it fits (cfg3),
// L2-resident global memory otherwise (cfg4, cfg5).
// Alg. 1 lines 16-25 per route; per-chunk maps start -> (end, hits) go to the
// workspace; the last CTA joins them along q0's path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "kernels_common.cuh"

namespace parem {

namespace {

constexpr uint32_t kMaxGroups = 32;

__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

struct LanesSmem {
    size_t tab, lcnt, grp, flag, total;
};

__host__ __device__ __forceinline__ LanesSmem lanes_layout(const DevDfa& d, bool smem_tab) {
    LanesSmem s;
    const size_t ES = d.lanes_u32 ? 4 : 2;
    size_t o = 0;
    // the table is placed at a shared address that is a multiple of its column stride
    // (Qpad * ES) so the base can be OR-ed into column offsets; reserve that much slack
    s.tab = o;  o = al16(o + (smem_tab ? (size_t)d.Apad * d.Qpad * ES + (size_t)d.Qpad * ES : 0));
    s.lcnt = o; o = al16(o + 4 * (size_t)(d.A + 1));
    s.grp = o;  o = al16(o + 16 * (size_t)kMaxGroups);   // per group: b0, b1
    s.flag = o; o = al16(o + 32);
    s.total = o;
    return s;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Warp-cooperative boundary_of(): one warp scans the snap window and takes the first
// position of the minimum |L(T[b-1])| (same function as the serial version).
__device__ __forceinline__ uint64_t boundary_warp(const MatchParams& P, uint64_t i, const uint32_t* Lcnt,
                                                  uint32_t lane) {
    if (i == 0) return 0;
    if (i >= P.p) return P.n;
    const uint64_t x = i * P.L;
    if (P.policy != PAREM_BOUNDARY_SNAP || P.win == 0) return x;
    uint64_t hi = x + P.win;
    if (hi > P.n - 1) hi = P.n - 1;
    unsigned long long best = ~0ull;
    for (uint64_t y = x + lane; y <= hi; y += 32) {
        const uint32_t c = __ldg(P.in + y - 1);
        const unsigned long long k = c < P.d.A ? Lcnt[c] : 0xFFFFFFFEull;
        const unsigned long long key = (k << 32) | (unsigned long long)(y - x);
        best = key < best ? key : best;
    }
    best = warp_min_u64(best);
    return x + (best & 0xFFFFFFFFull);
}

template <int U, bool SMEM, bool W32>
__global__ void __launch_bounds__(1024) lanes_kernel(const MatchParams P) {
    using ET = typename std::conditional<W32, uint32_t, uint16_t>::type;
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t A = d.A, Qpad = d.Qpad;
    const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u;
    const uint32_t Tg = P.tg, G = T / Tg, g = tid / Tg, gt = tid - g * Tg, gw = gt >> 5;
    const LanesSmem Ly = lanes_layout(d, SMEM);
    uint32_t* Lcnt = reinterpret_cast<uint32_t*>(sm + Ly.lcnt);
    unsigned long long* grp = reinterpret_cast<unsigned long long*>(sm + Ly.grp);
    uint32_t* flag = reinterpret_cast<uint32_t*>(sm + Ly.flag);
    constexpr uint32_t ES = W32 ? 4 : 2, ACC = W32 ? 31 : 15;

    // shared address of the staged table, aligned to the column stride Qpad*ES
    const uint32_t COLSTRIDE = Qpad * ES;
    const uint32_t sraw = static_cast<uint32_t>(__cvta_generic_to_shared(sm + Ly.tab));
    const uint32_t sbase = (sraw + COLSTRIDE - 1) / COLSTRIDE * COLSTRIDE;
    if (SMEM) {   // stage the symbol-major table (A1 product) into shared memory
        const size_t bytes = (size_t)d.Apad * Qpad * ES;
        const uint4* src = reinterpret_cast<const uint4*>(d.lanes_tab);
        uint4* dst = reinterpret_cast<uint4*>(sm + Ly.tab + (sbase - sraw));
        for (size_t i = tid; i < bytes / 16; i += T) dst[i] = __ldg(src + i);
    }
    for (uint32_t i = tid; i <= A; i += T) Lcnt[i] = __ldg(d.Lcnt + i);
    __syncthreads();

    // ---- A2: boundaries of this group's chunk (its first warp scans the snap windows) ----
    const uint64_t t = (uint64_t)blockIdx.x * G + g;
    const bool live = t < P.p;
    if (live && gw == 0) {
        const uint64_t b0 = boundary_warp(P, t, Lcnt, lane);
        const uint64_t b1 = boundary_warp(P, t + 1, Lcnt, lane);
        if (lane == 0) {
            grp[2 * g] = b0;
            grp[2 * g + 1] = b1;
        }
    }
    __syncthreads();
    uint64_t b0 = 0, b1 = 0;
    uint32_t cnt = 0, q0 = 0, rc = 0;
    const uint32_t* list = nullptr;
    if (live) {
        b0 = grp[2 * g];
        b1 = grp[2 * g + 1];
        if (t == 0) {
            bool dead;
            q0 = start_state(P, &dead);
            cnt = 1;
            rc = 1;
        } else {
            const uint32_t c = P.in[b0 - 1];
            const uint32_t li = (P.cand == PAREM_CANDIDATES_ENUM || c >= A) ? A : c;
            cnt = Lcnt[li];
            list = d.Llist + __ldg(d.Loff + li);
            rc = route_count(P, c, P.in[b0], cnt);
        }
    }

    // table offsets: next = (e & SMASK) | col, col = c * COLSTRIDE (+ the shared base)
    const unsigned char* gtab = reinterpret_cast<const unsigned char*>(d.lanes_tab);
    const uint32_t SMASK = (Qpad - 1u) * ES;
    const uint32_t CMASK = d.Apad - 1u;   // keeps invalid bytes (ESYMBOL) inside the table
    const uint32_t cbase = SMEM ? sbase : 0u;
    uint32_t* mend = reinterpret_cast<uint32_t*>(P.maps);
    uint32_t* mhits = P.map_hits;
    uint32_t bad = 0;

    // ---- A3: every pass advances up to Tg*U candidates over the whole chunk ----
    for (uint32_t base = 0; base < cnt; base += Tg * U) {
        uint32_t e[U], h[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t k = base + gt + (uint32_t)u * Tg;
            const uint32_t s = k < cnt ? (t == 0 ? q0 : __ldg(list + k)) : 0u;
            e[u] = s * ES;
            h[u] = 0;
        }
        const bool warp_active = base + gw * 32u < cnt;
        const bool check = (base == 0) && (gw == 0);   // one warp validates the bytes once
        if (warp_active) {
            auto lookup = [&](uint32_t col) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t off = (e[u] & SMASK) | col;
                    uint32_t v;
                    if constexpr (SMEM) {
                        // col already carries the table's shared base (disjoint from SMASK bits)
                        if constexpr (W32) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(off));
                        else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(off));
                    } else {
                        v = __ldg(reinterpret_cast<const ET*>(gtab + off));
                    }
                    e[u] = v;
                    h[u] += v >> ACC;
                }
            };
            auto step = [&](uint32_t c) { lookup((c & CMASK) * COLSTRIDE + cbase); };
            // byte k of w -> its column offset: PRMT (+ LOP3 when A < 256) + IMAD, shared by
            // the U routes of this thread
            auto step_w = [&](uint32_t w, uint32_t k) {
                uint32_t c = __byte_perm(w, 0u, 0x4440u | k);
                if (A < 256) c &= CMASK;
                lookup(c * COLSTRIDE + cbase);
            };
            uint64_t a = b0;
            const uint64_t mis = (uint64_t)(((uintptr_t)(P.in + a)) & 15u);
            uint64_t head = mis ? a + (16 - mis) : a;
            if (head > b1) head = b1;
            for (; a < head; ++a) {
                const uint32_t c = P.in[a];
                if (check && c >= A) bad = 1;
                step(c);
            }
            const uint32_t nvec = (uint32_t)((b1 - a) >> 4);
            const uint8_t* p = P.in + a;
            for (uint32_t v = 0; v < nvec; ++v) {
                const uint4 x = ldg_v4(p + 16ull * v);
                if (check) bad |= badbits(x.x, A) | badbits(x.y, A) | badbits(x.z, A) | badbits(x.w, A);
                const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    step_w(w4[q], 0);
                    step_w(w4[q], 1);
                    step_w(w4[q], 2);
                    step_w(w4[q], 3);
                }
            }
            a += (uint64_t)nvec << 4;
            for (; a < b1; ++a) {
                const uint32_t c = P.in[a];
                if (check && c >= A) bad = 1;
                step(c);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t k = base + gt + (uint32_t)u * Tg;
            if (k < cnt) {
                const uint32_t s = t == 0 ? q0 : __ldg(list + k);
                const uint64_t r = t * (uint64_t)Qpad + s;
                mend[r] = (e[u] & SMASK) / ES;
                mhits[r] = h[u];
            }
        }
    }
    if (live && gt == 0) {
        atomicAdd(&P.hdr->routes, (unsigned long long)rc);
        atomicAdd(&P.hdr->steps, (unsigned long long)rc * (b1 - b0));
        if (cnt == 0 && first_bad(P.in, b0, b1, A) < b1) bad = 1;   // R_i empty: still validate
    }
    if (live && gt == 0 && bad) {
        const uint64_t off = first_bad(P.in, b0, b1, A);
        if (off < b1) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
    }

    // ---- last-CTA detection, then A4/A5: the join along q0's path ----
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&P.hdr->done, 1u);
        *flag = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    if (tid == 0) {
        bool dead;
        uint32_t q = start_state(P, &dead);
        unsigned long long hits = 0;
        if (!dead) {
            for (uint64_t i = 0; i < P.p; ++i) {
                if (d.has_sink && q == d.sink) break;   // DEAD is absorbing (C9)
                const uint64_t r = i * Qpad + q;
                const uint32_t ne = ld_cg_u32(mend + r);
                hits += ld_cg_u32(mhits + r);
                q = ne;
            }
        }
        write_result(P, q, hits, dead);
    }
}

template <int U, bool SMEM, bool W32>
const void* lanes_fn() {
    return reinterpret_cast<const void*>(&lanes_kernel<U, SMEM, W32>);
}

const void* lanes_dispatch(uint32_t U, bool smem, bool w32) {
#define PAREM_LANES(SM_, W_)                              \
    switch (U) {                                          \
        case 1: return lanes_fn<1, SM_, W_>();            \
        case 2: return lanes_fn<2, SM_, W_>();            \
        case 3: return lanes_fn<3, SM_, W_>();            \
        case 4: return lanes_fn<4, SM_, W_>();            \
        case 6: return lanes_fn<6, SM_, W_>();            \
        case 8: return lanes_fn<8, SM_, W_>();            \
        default: return nullptr;                          \
    }
    if (smem && !w32) { PAREM_LANES(true, false) }
    if (smem && w32) { PAREM_LANES(true, true) }
    if (!smem && !w32) { PAREM_LANES(false, false) }
    if (!smem && w32) { PAREM_LANES(false, true) }
#undef PAREM_LANES
    return nullptr;
}

}  // namespace

uint32_t lanes_max_groups() { return kMaxGroups; }

size_t lanes_smem_bytes(const DevDfa& d, bool smem_tab) { return lanes_layout(d, smem_tab).total; }

int lanes_blocks_per_sm(uint32_t U, bool smem_tab, bool u32, uint32_t threads, size_t smem) {
    const void* fn = lanes_dispatch(U, smem_tab, u32);
    if (!fn) return 0;
    smem_optin(fn, smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, (int)threads, smem) != cudaSuccess) return 0;
    return nb;
}

int launch_lanes(const Plan& plan, const MatchParams& P, cudaStream_t s) {
    const void* fn = lanes_dispatch(plan.U, plan.smem_tab != 0, P.d.lanes_u32 != 0);
    if (!fn) {
        set_error("no lanes kernel for U=%u", plan.U);
        return PAREM_EINTERNAL;
    }
    cudaError_t e = smem_optin(fn, plan.smem);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    void* args[] = {const_cast<MatchParams*>(&P)};
    e = cudaLaunchKernel(fn, dim3((unsigned)plan.grid), dim3(plan.threads), args, plan.smem, s);
    if (e != cudaSuccess) {
        set_error("lanes kernel launch: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    prof_after("lanes", s);
    return PAREM_OK;
}

}  // namespace parem
