// kernels_lanes.cu -- multi-start chunk simulation for large DFAs (internal states > 32):
// one CTA per chunk, the chunk's candidate start states R_i spread over the CTA's lanes
// (U per thread for ILP), all lanes consuming the SAME byte each step (broadcast 16-byte
// loads) so step k's lookups all hit column T[k] of the symbol-major table -- shared
// memory when it fits (cfg3), L2-resident global memory otherwise (cfg4, cfg5).
// Alg. 1 lines 16-25 per route; per-chunk maps start -> (end, hits) go to the
// workspace; the last CTA joins them along q0's path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "kernels_common.cuh"

namespace parem {

namespace {

__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

struct LanesSmem {
    size_t tab, lcnt, red, flag, total;
};

__host__ __device__ __forceinline__ LanesSmem lanes_layout(const DevDfa& d, bool smem_tab) {
    LanesSmem s;
    const size_t ES = d.lanes_u32 ? 4 : 2;
    size_t o = 0;
    s.tab = o;  o = al16(o + (smem_tab ? (size_t)d.Apad * d.Qpad * ES : 0));
    s.lcnt = o; o = al16(o + 4 * (size_t)(d.A + 1));
    s.red = o;  o = al16(o + 8 * 32);
    s.flag = o; o = al16(o + 32);
    s.total = o;
    return s;
}

__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, unsigned long long* red) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = w < v ? w : v;
    }
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long m = ~0ull;
    for (uint32_t i = 0; i < nw; ++i) m = red[i] < m ? red[i] : m;
    __syncthreads();
    return m;
}

// Cooperative version of boundary_of(): the CTA scans the snap window in parallel and
// takes the first position of the minimum |L(T[b-1])| (same function as the serial one).
__device__ __forceinline__ uint64_t boundary_cta(const MatchParams& P, uint64_t i, const uint32_t* Lcnt,
                                                 unsigned long long* red) {
    if (i == 0) return 0;
    if (i >= P.p) return P.n;
    const uint64_t x = i * P.L;
    if (P.policy != PAREM_BOUNDARY_SNAP || P.win == 0) return x;
    uint64_t hi = x + P.win;
    if (hi > P.n - 1) hi = P.n - 1;
    unsigned long long best = ~0ull;
    for (uint64_t y = x + threadIdx.x; y <= hi; y += blockDim.x) {
        const uint32_t c = __ldg(P.in + y - 1);
        const unsigned long long k = c < P.d.A ? Lcnt[c] : 0xFFFFFFFEull;
        const unsigned long long key = (k << 32) | (unsigned long long)(y - x);
        best = key < best ? key : best;
    }
    best = block_min_u64(best, red);
    return x + (best & 0xFFFFFFFFull);
}

template <int U, bool SMEM, bool W32>
__global__ void __launch_bounds__(1024) lanes_kernel(const MatchParams P) {
    using ET = typename std::conditional<W32, uint32_t, uint16_t>::type;
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t A = d.A, Qpad = d.Qpad;
    const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
    const LanesSmem Ly = lanes_layout(d, SMEM);
    uint32_t* Lcnt = reinterpret_cast<uint32_t*>(sm + Ly.lcnt);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(sm + Ly.red);
    uint32_t* flag = reinterpret_cast<uint32_t*>(sm + Ly.flag);
    constexpr uint32_t ES = W32 ? 4 : 2, ACC = W32 ? 31 : 15;

    if (SMEM) {   // stage the symbol-major table (A1 product) into shared memory
        const size_t bytes = (size_t)d.Apad * Qpad * ES;
        const uint4* src = reinterpret_cast<const uint4*>(d.lanes_tab);
        uint4* dst = reinterpret_cast<uint4*>(sm + Ly.tab);
        for (size_t i = tid; i < bytes / 16; i += T) dst[i] = __ldg(src + i);
    }
    for (uint32_t i = tid; i <= A; i += T) Lcnt[i] = __ldg(d.Lcnt + i);
    __syncthreads();

    // ---- A2: boundaries and R_i of this CTA's chunk ----
    const uint64_t t = blockIdx.x;
    const uint64_t b0 = boundary_cta(P, t, Lcnt, red);
    const uint64_t b1 = boundary_cta(P, t + 1, Lcnt, red);
    uint32_t cnt, q0 = 0, rc;
    const uint32_t* list = nullptr;
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

    const unsigned char* tab = SMEM ? (sm + Ly.tab) : reinterpret_cast<const unsigned char*>(d.lanes_tab);
    const uint32_t SH = d.log2Qpad + (W32 ? 2 : 1);
    const uint32_t SMASK = (Qpad - 1u) * ES;
    const uint32_t CMASK = d.Apad - 1u;
    uint32_t* mend = reinterpret_cast<uint32_t*>(P.maps);
    uint32_t* mhits = P.map_hits;
    uint32_t bad = 0;

    // ---- A3: every pass advances up to T*U candidates over the whole chunk ----
    for (uint32_t base = 0; base < cnt; base += T * U) {
        uint32_t e[U], h[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t k = base + tid + (uint32_t)u * T;
            const uint32_t s = k < cnt ? (t == 0 ? q0 : __ldg(list + k)) : 0u;
            e[u] = s * ES;
            h[u] = 0;
        }
        const bool warp_active = base + warp * 32u < cnt;
        const bool check = (base == 0) && (warp == 0);   // one warp validates the bytes once
        if (warp_active) {
            auto step = [&](uint32_t c) {
                const uint32_t col = (c & CMASK) << SH;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t off = (e[u] & SMASK) | col;
                    uint32_t v;
                    if (SMEM) v = *reinterpret_cast<const ET*>(tab + off);
                    else v = __ldg(reinterpret_cast<const ET*>(tab + off));
                    e[u] = v;
                    h[u] += v >> ACC;
                }
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
            const uint64_t nvec = (b1 - a) >> 4;
            const uint8_t* p = P.in + a;
            for (uint64_t v = 0; v < nvec; ++v) {
                const uint4 x = ldg_v4(p + 16 * v);
                if (check) bad |= badbits(x.x, A) | badbits(x.y, A) | badbits(x.z, A) | badbits(x.w, A);
                const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    step(w4[q] & 0xFFu);
                    step((w4[q] >> 8) & 0xFFu);
                    step((w4[q] >> 16) & 0xFFu);
                    step(w4[q] >> 24);
                }
            }
            a += nvec << 4;
            for (; a < b1; ++a) {
                const uint32_t c = P.in[a];
                if (check && c >= A) bad = 1;
                step(c);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t k = base + tid + (uint32_t)u * T;
            if (k < cnt) {
                const uint32_t s = t == 0 ? q0 : __ldg(list + k);
                const uint64_t r = t * (uint64_t)Qpad + s;
                mend[r] = (e[u] & SMASK) / ES;
                mhits[r] = h[u];
            }
        }
    }
    if (tid == 0) {
        atomicAdd(&P.hdr->routes, (unsigned long long)rc);
        atomicAdd(&P.hdr->steps, (unsigned long long)rc * (b1 - b0));
    }
    if (cnt == 0 && tid == 0 && first_bad(P.in, b0, b1, A) < b1) bad = 1;   // R_i empty: still validate
    if (warp == 0 && lane == 0 && bad) {
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
        case 4: return lanes_fn<4, SM_, W_>();            \
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

uint32_t lanes_round_u(uint32_t u) { return u <= 1 ? 1 : u <= 2 ? 2 : u <= 4 ? 4 : 8; }

size_t lanes_smem_bytes(const DevDfa& d, bool smem_tab) { return lanes_layout(d, smem_tab).total; }

int lanes_blocks_per_sm(uint32_t U, bool smem_tab, bool u32, uint32_t threads, size_t smem) {
    const void* fn = lanes_dispatch(U, smem_tab, u32);
    if (!fn) return 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
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
    return PAREM_OK;
}

}  // namespace parem
