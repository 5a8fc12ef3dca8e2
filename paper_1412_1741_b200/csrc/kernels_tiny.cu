// kernels_tiny.cu -- multi-start chunk simulation for small DFAs (internal states <= 32):
// one THREAD per chunk, the chunk's candidate start states R_i as K registers that all
// advance in one pass over the chunk's bytes (Alg. 1 lines 16-25), dense
// per-chunk maps start -> (end, hits) composed by warps, and a
// last-CTA fold of the per-CTA tile maps along q0's path.
//
// Lookup tables in shared memory:
//   * for A <= 4 a 4-bit-group STRIDE table: one lookup advances a route by KS = 4/B
//     symbols (B = bits per symbol), entry = dest << 11 | lane << 2 | hits << 28, replicated
//     per lane so lane l always reads bank l (conflict-free); the next lookup's byte
//     offset is (e & 0xFFFF) | group << 7 -- one LOP3, one LDS, one shift-add per group;
//   * tab1[s][c] = dest | acc << 15 for single-symbol steps (unaligned heads/tails) and
//     for the generic path (A > 4).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels_common.cuh"

namespace parem {

namespace {

constexpr uint32_t kT = kTinyThreads;
constexpr uint32_t kWarps = kT / 32;

__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

struct TinySmem {
    size_t tabk, tab1, lcnt, loff, llist, mend, mhits, wend, whits, flag, total;
};

__host__ __device__ __forceinline__ TinySmem tiny_layout(uint32_t Qp, uint32_t Qpad, uint32_t A, uint32_t Lsum_all,
                                                         uint32_t B) {
    TinySmem s;
    size_t o = 0;
    s.tabk = o;  o += B ? (size_t)Qp * 2048 : 0;
    s.tab1 = o;  o = al16(o + (size_t)Qp * A * 2);
    s.lcnt = o;  o = al16(o + 4 * (size_t)(A + 1));
    s.loff = o;  o = al16(o + 4 * (size_t)(A + 1));
    s.llist = o; o = al16(o + 4 * (size_t)Lsum_all);
    s.mend = o;  o = al16(o + (size_t)kT * Qpad);
    s.mhits = o; o = al16(o + 4 * (size_t)kT * Qpad);
    s.wend = o;  o = al16(o + 4 * (size_t)kWarps * Qpad);
    s.whits = o; o = al16(o + 8 * (size_t)kWarps * Qpad);
    s.flag = o;  o = al16(o + 16);
    s.total = o;
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

    __device__ __forceinline__ void group(uint32_t g7, const unsigned char* __restrict__ tabk) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
            e[j] = *reinterpret_cast<const uint32_t*>(tabk + ((e[j] & 0xFFFFu) | g7));
            h[j] += e[j] >> 28;
        }
    }

    // four symbols packed in one little-endian word
    __device__ __forceinline__ void word(uint32_t w, const unsigned char* __restrict__ tabk,
                                         const uint16_t* __restrict__ tab1, uint32_t A, uint32_t badmask,
                                         uint32_t lane4) {
        if constexpr (B == 2) {
            bad |= w & badmask;
            // b0 | b1<<2 | b2<<4 | b3<<6 lands in bits 24..31 of the product (no carries:
            // every cross term occupies its own 2-bit slot below bit 24 or above bit 31)
            const uint32_t P = w * 0x01041040u;
            group((P >> 17) & 0x780u, tabk);    // symbols 0,1
            group((P >> 21) & 0x780u, tabk);    // symbols 2,3
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

    // advance every route over in[a, b)
    __device__ __forceinline__ void walk(const uint8_t* __restrict__ in, uint64_t a, uint64_t b,
                                         const unsigned char* __restrict__ tabk, const uint16_t* __restrict__ tab1,
                                         uint32_t A, uint32_t badmask, uint32_t lane4) {
        const uint64_t mis = (uint64_t)(((uintptr_t)(in + a)) & 15u);
        uint64_t head = mis ? a + (16 - mis) : a;
        if (head > b) head = b;
        for (; a < head; ++a) step1(in[a], tab1, A, lane4);
        uint64_t nvec = (b - a) >> 4;
        const uint8_t* p = in + a;
#pragma unroll 2
        for (uint64_t v = 0; v < nvec; ++v) {
            const uint4 x = ldg_v4(p + 16 * v);
            word(x.x, tabk, tab1, A, badmask, lane4);
            word(x.y, tabk, tab1, A, badmask, lane4);
            word(x.z, tabk, tab1, A, badmask, lane4);
            word(x.w, tabk, tab1, A, badmask, lane4);
        }
        a += nvec << 4;
        for (; a < b; ++a) step1(in[a], tab1, A, lane4);
    }
};

template <int K, int B>
__global__ void __launch_bounds__(kT) tiny_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t Qp = d.Qp, Qpad = d.Qpad, A = d.A;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const TinySmem L = tiny_layout(Qp, Qpad, A, d.Lsum_all, B);
    uint32_t* tabk32 = reinterpret_cast<uint32_t*>(sm + L.tabk);
    uint16_t* tab1 = reinterpret_cast<uint16_t*>(sm + L.tab1);
    uint32_t* Lcnt = reinterpret_cast<uint32_t*>(sm + L.lcnt);
    uint32_t* Loff = reinterpret_cast<uint32_t*>(sm + L.loff);
    uint32_t* Llist = reinterpret_cast<uint32_t*>(sm + L.llist);
    uint8_t* mend = sm + L.mend;
    uint32_t* mhits = reinterpret_cast<uint32_t*>(sm + L.mhits);
    uint32_t* wend = reinterpret_cast<uint32_t*>(sm + L.wend);
    unsigned long long* whits = reinterpret_cast<unsigned long long*>(sm + L.whits);
    uint32_t* flag = reinterpret_cast<uint32_t*>(sm + L.flag);

    // ---- stage the tables (A1 products) into shared memory ----
    if (B)
        for (uint32_t i = tid; i < Qp * 512u; i += kT) tabk32[i] = __ldg(d.stride + (i >> 5)) | ((i & 31u) << 2);
    for (uint32_t i = tid; i < Qp * A; i += kT) tab1[i] = __ldg(d.tab1 + i);
    for (uint32_t i = tid; i <= A; i += kT) {
        Lcnt[i] = __ldg(d.Lcnt + i);
        Loff[i] = __ldg(d.Loff + i);
    }
    for (uint32_t i = tid; i < d.Lsum_all; i += kT) Llist[i] = __ldg(d.Llist + i);
    for (uint32_t q = 0; q < Qpad; ++q) {      // identity map: non-candidates keep their state
        mend[tid * Qpad + q] = (uint8_t)q;
        mhits[tid * Qpad + q] = 0;
    }
    __syncthreads();

    // ---- A2 + A3: this thread's chunk, its R_i, one pass advancing all candidates ----
    const uint64_t t = (uint64_t)blockIdx.x * kT + tid;
    uint32_t rc = 0;
    unsigned long long steps = 0;
    if (t < P.p) {
        const uint64_t b0 = boundary_of(P, t, Lcnt), b1 = boundary_of(P, t + 1, Lcnt);
        uint32_t cnt, loff = 0, q0 = 0;
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
        // per-byte invalid bits for A = 1, 2, 4 (power of two): every bit above log2(A)
        const uint32_t bm = B ? (0xFFu & ~(A - 1u)) * 0x01010101u : 0u;
        const uint32_t lane4 = lane << 2;
        uint32_t badacc = 0;
        for (uint32_t base = 0; base < cnt; base += K) {
            Routes<K, B> r;
            r.bad = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const uint32_t k = min(base + (uint32_t)j, cnt - 1);
                const uint32_t s = t == 0 ? q0 : Llist[loff + k];
                r.e[j] = B ? ((s << 11) | lane4) : s;
                r.h[j] = 0;
            }
            r.walk(P.in, b0, b1, sm + L.tabk, tab1, A, bm, lane4);
            badacc |= r.bad;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                if (base + (uint32_t)j < cnt) {
                    const uint32_t s = t == 0 ? q0 : Llist[loff + base + j];
                    mend[tid * Qpad + s] = (uint8_t)r.state(j);
                    mhits[tid * Qpad + s] = r.h[j];
                }
            }
        }
        steps = (unsigned long long)rc * (b1 - b0);
        if (cnt == 0 && first_bad(P.in, b0, b1, A) < b1) badacc = 1;   // R_i empty: still validate
        if (badacc) {
            const uint64_t off = first_bad(P.in, b0, b1, A);
            if (off < b1) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
        }
    }

    // ---- stats (block reduce -> 2 atomics per CTA) ----
    {
        const uint32_t rs = warp_sum(rc);
        const unsigned long long ss = warp_sum(steps);
        if (lane == 0) {
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
        const uint32_t me = (uint32_t)(m & 0xFFu);
        const unsigned long long mh = m >> 8;
        const uint32_t ne = __shfl_sync(0xFFFFFFFFu, me, ce);
        const unsigned long long nh = __shfl_sync(0xFFFFFFFFu, mh, ce);
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

template <int K, int B>
const void* tiny_fn() {
    return reinterpret_cast<const void*>(&tiny_kernel<K, B>);
}

const void* tiny_dispatch(uint32_t K, uint32_t B) {
#define PAREM_TINY_B(BB)                      \
    switch (K) {                              \
        case 1: return tiny_fn<1, BB>();      \
        case 2: return tiny_fn<2, BB>();      \
        case 3: return tiny_fn<3, BB>();      \
        case 4: return tiny_fn<4, BB>();      \
        case 6: return tiny_fn<6, BB>();      \
        case 8: return tiny_fn<8, BB>();      \
        case 12: return tiny_fn<12, BB>();    \
        case 16: return tiny_fn<16, BB>();    \
        case 32: return tiny_fn<32, BB>();    \
        default: return nullptr;              \
    }
    if (B == 0) { PAREM_TINY_B(0) }
    if (B == 1) { PAREM_TINY_B(1) }
    if (B == 2) { PAREM_TINY_B(2) }
#undef PAREM_TINY_B
    return nullptr;
}

}  // namespace

uint32_t tiny_round_slots(uint32_t k) {
    static const uint32_t ks[] = {1, 2, 3, 4, 6, 8, 12, 16, 32};
    for (uint32_t v : ks)
        if (k <= v) return v;
    return 32;
}

size_t tiny_smem_bytes(const DevDfa& d, uint32_t B) { return tiny_layout(d.Qp, d.Qpad, d.A, d.Lsum_all, B).total; }

int tiny_blocks_per_sm(uint32_t K, uint32_t B, size_t smem) {
    const void* fn = tiny_dispatch(K, B);
    if (!fn) return 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kT, smem) != cudaSuccess) return 0;
    return nb;
}

int launch_tiny(const Plan& plan, const MatchParams& P, cudaStream_t s) {
    const void* fn = tiny_dispatch(plan.slots, P.d.sym_bits);
    if (!fn) {
        set_error("no tiny kernel for K=%u B=%u", plan.slots, P.d.sym_bits);
        return PAREM_EINTERNAL;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    void* args[] = {const_cast<MatchParams*>(&P)};
    e = cudaLaunchKernel(fn, dim3((unsigned)plan.grid), dim3(kT), args, plan.smem, s);
    if (e != cudaSuccess) {
        set_error("tiny kernel launch: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    return PAREM_OK;
}

}  // namespace parem
