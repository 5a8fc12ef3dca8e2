// kernels_find.cu -- SURVEY §8(f) NEXT-4: match END positions.  Alg. 1 keeps a visited-state
// vector Rr per route; the positions of the matches are the steps whose state is
// in F.  After a match has produced its per-chunk maps (tiny / lanes kernels) or the true
// boundary states (converging path), every chunk's entering state q_i and hit count h_i are
// resolved, h is exclusive-scanned into output offsets, and every chunk is walked ONCE more
// from q_i -- one route per chunk, no speculation -- writing the offsets k (q_{k+1} in F) of
// its matches to out[base_i + j] (ascending overall; at most max_positions are written).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels_common.cuh"

namespace parem {

namespace {

constexpr uint32_t kFindThreads = 256;
constexpr uint32_t kScanBlock = 1024;   // chunks per scan block (one CTA, 4 per thread)
constexpr uint32_t kGroup = 32;         // tiny path: chunks per composed group

// chunk boundaries exactly as the match computed them
__device__ __forceinline__ uint64_t find_b(const MatchParams& P, uint64_t i) {
    return boundary_of(P, i, P.d.Lcnt);
}

// ---- tiny path: compose groups of 32 chunk maps (lane q = start state q) ----
__global__ void __launch_bounds__(kFindThreads) find_group_kernel(const MatchParams P, uint64_t groups) {
    const uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u, Qpad = P.d.Qpad;
    if (g >= groups) return;
    uint32_t ce = lane < Qpad ? lane : 0;
    unsigned long long ch = 0;
    const uint64_t lo = g * kGroup, hi = min(P.p, lo + kGroup);
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t r = i * Qpad + ce;
        ch += P.fmhits[r];
        ce = P.fmend[r];
    }
    if (lane < Qpad) {
        P.fgend[g * Qpad + lane] = ce;
        P.fghits[g * Qpad + lane] = ch;
    }
}

// ---- tiny path: super-groups of 32 groups (1024 chunks): warp per super-group composes its
// group maps (lane = state) into a super map (end only), then ONE warp walks the super maps
// along q0's path, then every super-group's warp walks its 32 groups from its entering state
__global__ void __launch_bounds__(kFindThreads) find_super_kernel(const MatchParams P, uint64_t groups) {
    const uint64_t sg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u, Qpad = P.d.Qpad;
    const uint64_t nsg = (groups + 31) / 32;
    if (sg >= nsg) return;
    uint32_t ce = lane < Qpad ? lane : 0;
    const uint64_t lo = sg * 32, hi = min(groups, lo + 32);
    for (uint64_t g = lo; g < hi; ++g) ce = P.fgend[g * Qpad + ce];
    if (lane < Qpad) P.fsend[sg * Qpad + lane] = ce;
}

__global__ void find_group_seq_kernel(const MatchParams P, uint64_t groups) {
    const uint32_t lane = threadIdx.x & 31u, Qpad = P.d.Qpad;
    if (threadIdx.x >= 32) return;
    const uint64_t nsg = (groups + 31) / 32;
    bool dead;
    uint32_t q = start_state(P, &dead);
    for (uint64_t s0 = 0; s0 < nsg; s0 += 32) {   // the maps of 32 super-groups load at once
        uint32_t e[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) e[j] = (s0 + j < nsg && lane < Qpad) ? P.fsend[(s0 + j) * Qpad + lane] : 0u;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (s0 + j < nsg) {
                if (lane == 0) P.fsq[s0 + j] = q;
                q = __shfl_sync(0xFFFFFFFFu, e[j], q);
            }
    }
}

__global__ void __launch_bounds__(kFindThreads) find_group_in_kernel(const MatchParams P, uint64_t groups) {
    const uint64_t sg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nsg = (groups + 31) / 32;
    if (sg >= nsg || lane != 0) return;
    uint32_t q = P.fsq[sg];
    const uint64_t lo = sg * 32, hi = min(groups, lo + 32);
    for (uint64_t g = lo; g < hi; ++g) {
        P.fgq[g] = q;
        q = P.fgend[g * P.d.Qpad + q];
    }
}

// ---- tiny path: per chunk q_i and h_i, one thread per group walking its 32 chunk maps ----
__global__ void __launch_bounds__(kFindThreads) find_chunks_kernel(const MatchParams P, uint64_t groups) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= groups) return;
    const uint32_t Qpad = P.d.Qpad;
    uint32_t q = P.fgq[g];
    const uint64_t lo = g * kGroup, hi = min(P.p, lo + kGroup);
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t r = i * Qpad + q;
        P.fchunk_q[i] = q;
        P.fchunk_h[i] = P.fmhits[r];
        q = P.fmend[r];
    }
}

// ---- lanes path: one thread walks the p dense chunk maps (p is small on this path) ----
__global__ void find_lanes_seq_kernel(const MatchParams P) {
    if (threadIdx.x != 0) return;
    const uint32_t* mend = reinterpret_cast<const uint32_t*>(P.maps);
    bool dead;
    uint32_t q = start_state(P, &dead);
    for (uint64_t i = 0; i < P.p; ++i) {
        P.fchunk_q[i] = q;
        if (P.d.has_sink && q == P.d.sink) {   // dead: absorbing, no hits (C9); map rows of the
            P.fchunk_h[i] = 0;                 // sink are not written by the lanes kernel
            continue;
        }
        const uint64_t r = i * P.d.Qpad + q;
        P.fchunk_h[i] = P.map_hits[r];
        q = mend[r];
    }
}

// ---- exclusive scan of the per-chunk hit counts (u32) into u64 output offsets ----
__global__ void __launch_bounds__(kScanBlock / 4) find_scan_sums_kernel(const MatchParams P) {
    __shared__ unsigned long long ws[kScanBlock / 4 / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kScanBlock;
    unsigned long long s = 0;
    for (uint32_t k = 0; k < 4; ++k) {
        const uint64_t i = base + threadIdx.x * 4 + k;
        if (i < P.p) s += P.fchunk_h[i];
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (uint32_t w = 0; w < kScanBlock / 4 / 32; ++w) t += ws[w];
        P.fblock[blockIdx.x] = t;
    }
}

__global__ void find_scan_blocks_kernel(const MatchParams P, uint64_t nblocks) {
    if (threadIdx.x != 0) return;
    unsigned long long run = 0;
    for (uint64_t b = 0; b < nblocks; ++b) {
        const unsigned long long v = P.fblock[b];
        P.fblock[b] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(kScanBlock / 4) find_scan_apply_kernel(const MatchParams P) {
    __shared__ unsigned long long ws[kScanBlock / 4 / 32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kScanBlock;
    uint32_t v[4];
    unsigned long long s = 0;
    for (uint32_t k = 0; k < 4; ++k) {
        const uint64_t i = base + threadIdx.x * 4 + k;
        v[k] = i < P.p ? P.fchunk_h[i] : 0u;
        s += v[k];
    }
    // inclusive warp scan of the per-thread sums
    unsigned long long inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if ((int)lane >= o) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    unsigned long long woff = 0;
    for (uint32_t w = 0; w < warp; ++w) woff += ws[w];
    unsigned long long run = P.fblock[blockIdx.x] + woff + inc - s;
    for (uint32_t k = 0; k < 4; ++k) {
        const uint64_t i = base + threadIdx.x * 4 + k;
        if (i < P.p) P.fchunk_base[i] = run;
        run += v[k];
    }
}

// ---- emit: walk every chunk once from its true entering state ----
// tiny tables: tab1[s][c] = dest | acc(dest) << 15 (u16), staged in shared memory
__global__ void __launch_bounds__(kFindThreads) find_emit_tiny_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    uint16_t* tab = reinterpret_cast<uint16_t*>(sm);
    for (uint32_t i = threadIdx.x; i < d.Qp * d.A; i += blockDim.x) tab[i] = __ldg(d.tab1 + i);
    __syncthreads();
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.p) return;
    const uint64_t b0 = find_b(P, t), b1 = find_b(P, t + 1);
    uint32_t s = P.fchunk_q[t];
    unsigned long long o = P.fchunk_base[t];
    const uint32_t A = d.A;
    auto step = [&](uint32_t c, uint64_t k) {
        const uint32_t e = tab[s * A + (c < A ? c : A - 1)];
        s = e & 0x7FFFu;
        const uint32_t h = e >> 15;   // predicated store (see find_emit_lanes_kernel)
        if (h && o < P.fmax) P.fout[o] = k;
        o += h;
    };
    uint64_t a = b0;
    for (; a < b1 && (((uintptr_t)(P.in + a)) & 15u); ++a) step(P.in[a], a);
    uint4 nx = a + 16 <= b1 ? ldg_v4_na(P.in + a) : make_uint4(0, 0, 0, 0);
    for (; a + 16 <= b1; a += 16) {
        const uint4 x = nx;
        if (a + 32 <= b1) nx = ldg_v4_na(P.in + a + 16);
        const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) step(__byte_perm(w4[q], 0u, 0x4440u | k), a + 4 * q + k);
    }
    for (; a < b1; ++a) step(P.in[a], a);
}

// tiny tables with a stride table (A <= 4: B = 1 or 2 bits per symbol): one lookup per 4 / B
// symbols, the tiny kernel's lane-replicated layout (entry = dest << 11 | lane << 2 |
// hits << 28, lane l reads bank l).  A group with hits > 0 (rare for a search automaton) is
// re-walked symbol by symbol through tab1 to emit its positions.  ~1 LOP3 + 1 LDS per group
// instead of ~7 ops per symbol: the emit pass streams its chunk at close to the load rate.
template <int B>
__global__ void __launch_bounds__(kFindThreads) find_emit_stride_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t* tabk32 = reinterpret_cast<uint32_t*>(sm);
    uint16_t* tab1 = reinterpret_cast<uint16_t*>(sm + (size_t)d.Qp * 2048);
    for (uint32_t i = threadIdx.x; i < d.Qp * 512u; i += blockDim.x) tabk32[i] = __ldg(d.stride + (i >> 5)) | ((i & 31u) << 2);
    for (uint32_t i = threadIdx.x; i < d.Qp * d.A; i += blockDim.x) tab1[i] = __ldg(d.tab1 + i);
    __syncthreads();
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.p) return;
    const unsigned char* tabk = sm;
    const uint64_t b0 = find_b(P, t), b1 = find_b(P, t + 1);
    const uint32_t A = d.A, lane4 = lane << 2;
    uint32_t s = P.fchunk_q[t];
    unsigned long long o = P.fchunk_base[t];
    auto emit = [&](uint64_t k) {
        if (o < P.fmax) P.fout[o] = k;
        ++o;
    };
    auto step1 = [&](uint32_t c, uint64_t k) {
        const uint32_t e = tab1[s * A + (c < A ? c : A - 1)];
        s = e & 0x7FFFu;
        if (e >> 15) emit(k);
    };
    uint64_t a = b0;
    for (; a < b1 && (((uintptr_t)(P.in + a)) & 15u); ++a) step1(P.in[a], a);
    uint32_t e = (s << 11) | lane4;
    // one stride group: symbols (first, first + 1, ...) of word w, packed index g7
    auto group = [&](uint32_t g7, uint32_t w, uint32_t first, uint64_t pos) {
        const uint32_t prev = e;
        e = *reinterpret_cast<const uint32_t*>(tabk + ((e & 0xFFFFu) | g7));
        if (e >> 28) {   // rare: emit this group's positions symbol by symbol
            s = (prev & 0xFFFFu) >> 11;
#pragma unroll
            for (uint32_t j = 0; j < 4u / B; ++j) step1((w >> (8 * (first + j))) & 0xFFu, pos + j);
        }
    };
    auto word = [&](uint32_t w, uint64_t pos) {
        if constexpr (B == 2) {
            const uint32_t Pw = w * 130u;
            group(Pw & 0x780u, w, 0, pos);
            group(__umulhi(w, 0x00820000u) & 0x780u, w, 2, pos + 2);
        } else {
            const uint32_t Pw = w * 0x10204080u;
            group((Pw >> 21) & 0x780u, w, 0, pos);
        }
    };
    uint4 nx = a + 16 <= b1 ? ldg_v4_na(P.in + a) : make_uint4(0, 0, 0, 0);
    for (; a + 16 <= b1; a += 16) {
        const uint4 x = nx;
        if (a + 32 <= b1) nx = ldg_v4_na(P.in + a + 16);
        word(x.x, a);
        word(x.y, a + 4);
        word(x.z, a + 8);
        word(x.w, a + 12);
    }
    s = (e & 0xFFFFu) >> 11;
    for (; a < b1; ++a) step1(P.in[a], a);
}

// The same walk with the rows streamed by TMA (the default for GRID partitions): a
// thread-per-chunk 16-byte load stream costs 32 L1TEX wavefronts per warp request and the
// table's shared loads queue behind them (profiles/r02_ncu_find_emit*: 78 % short
// scoreboard); TMA boxes land in shared memory without that queue.  Warp w of the CTA owns
// 64 rows (lane l: rows l and l + 32, two chains); 64-row x 64-byte boxes, SWIZZLE_64B, two
// mbarrier stages; the remainder past the last full row (reading C7) is walked by its lane
// from global memory.
constexpr uint32_t kEBox = 64, kERows = 64, kEStages = 2, kEStage = kEBox * kERows, kEThreads = 512;

__host__ __device__ __forceinline__ size_t emit_tma_smem(const DevDfa& d) {
    return (((size_t)d.Qp * 2048 + (size_t)d.Qp * d.A * 2 + 1023) & ~(size_t)1023) +
           (kEThreads / 32) * (kEStages * kEStage + 8 * kEStages) + 1024;
}

template <int B>
__global__ void __launch_bounds__(kEThreads, 1) find_emit_stride_tma_kernel(const MatchParams P,
                                                                          const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t* tabk32 = reinterpret_cast<uint32_t*>(sm);
    uint16_t* tab1 = reinterpret_cast<uint16_t*>(sm + (size_t)d.Qp * 2048);
    const uint32_t sraw = smem_u32(sm);
    const uint32_t stg = (sraw + (uint32_t)((size_t)d.Qp * 2048 + (size_t)d.Qp * d.A * 2) + 1023u) & ~1023u;
    const uint32_t stage0 = stg + warp * kEStages * kEStage;
    const uint32_t mbar0 = stg + nw * kEStages * kEStage + warp * kEStages * 8u;
    const uint64_t row0 = (uint64_t)blockIdx.x * (nw * kERows) + warp * kERows;
    const uint32_t nst = (uint32_t)(P.L / kEBox);
    const bool warp_live = row0 < P.p;
    if (lane == 0 && warp_live) {
        for (uint32_t k = 0; k < kEStages; ++k) mbar_init(mbar0 + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t k = 0; k < kEStages && k < nst; ++k) {
            mbar_expect_tx(mbar0 + 8 * k, kEStage);
            tma_load_2d(stage0 + k * kEStage, &tmap, (int32_t)(k * kEBox), (int32_t)row0, mbar0 + 8 * k);
        }
    }
    for (uint32_t i = threadIdx.x; i < d.Qp * 512u; i += blockDim.x) tabk32[i] = __ldg(d.stride + (i >> 5)) | ((i & 31u) << 2);
    for (uint32_t i = threadIdx.x; i < d.Qp * d.A; i += blockDim.x) tab1[i] = __ldg(d.tab1 + i);
    __syncthreads();
    if (!warp_live) return;
    const unsigned char* tabk = sm;
    const uint32_t A = d.A, lane4 = lane << 2;
    const uint64_t ta = row0 + lane, tb = row0 + 32 + lane;
    const bool la = ta < P.p, lb = tb < P.p;
    uint32_t ea = ((la ? P.fchunk_q[ta] : 0u) << 11) | lane4, eb = ((lb ? P.fchunk_q[tb] : 0u) << 11) | lane4;
    unsigned long long oa = la ? P.fchunk_base[ta] : 0ull, ob = lb ? P.fchunk_base[tb] : 0ull;
    auto step1 = [&](uint32_t& s, unsigned long long& o, uint32_t c, uint64_t k) {
        const uint32_t e = tab1[s * A + (c < A ? c : A - 1)];
        s = e & 0x7FFFu;
        if (e >> 15) {
            if (o < P.fmax) P.fout[o] = k;
            ++o;
        }
    };
    // branch-free hot path: a vector's stride groups only OR their hit fields; a vector with
    // any hit is re-walked symbol by symbol from its entry state (rare for a search
    // automaton).  A branch per group would expose every lookup's latency.
    auto group = [&](uint32_t& e, uint32_t& hit, uint32_t g7) {
        e = *reinterpret_cast<const uint32_t*>(tabk + ((e & 0xFFFFu) | g7));
        hit |= e;
    };
    auto word = [&](uint32_t& e, uint32_t& hit, uint32_t w) {
        if constexpr (B == 2) {
            const uint32_t Pw = w * 130u;
            group(e, hit, Pw & 0x780u);
            group(e, hit, __umulhi(w, 0x00820000u) & 0x780u);
        } else {
            const uint32_t Pw = w * 0x10204080u;
            group(e, hit, (Pw >> 21) & 0x780u);
        }
    };
    auto rewalk = [&](uint32_t e0, unsigned long long& o, const uint4& v, uint64_t pos) {
        uint32_t s = (e0 & 0xFFFFu) >> 11;
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
        for (uint32_t q = 0; q < 4; ++q)
            for (uint32_t j = 0; j < 4; ++j) step1(s, o, (w4[q] >> (8 * j)) & 0xFFu, pos + 4 * q + j);
    };
    const uint32_t sw = (lane >> 1) & 3u, offa = lane * kEBox, offb = (lane + 32u) * kEBox;
    const uint64_t xa = ta * P.L, xb = tb * P.L;
    uint32_t slot = 0, phase = 0;
    for (uint32_t st = 0; st < nst; ++st) {
        mbar_wait(mbar0 + 8 * slot, phase);
        const uint32_t buf = stage0 + slot * kEStage;
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
            const uint32_t ou = (u ^ sw) << 4;
            const uint4 va = lds128(buf + offa + ou), vb = lds128(buf + offb + ou);
            const uint32_t ea0 = ea, eb0 = eb;
            uint32_t ha = 0, hb = 0;
            word(ea, ha, va.x);
            word(eb, hb, vb.x);
            word(ea, ha, va.y);
            word(eb, hb, vb.y);
            word(ea, ha, va.z);
            word(eb, hb, vb.z);
            word(ea, ha, va.w);
            word(eb, hb, vb.w);
            if (((ha | hb) >> 28) != 0) {
                if (la && (ha >> 28)) rewalk(ea0, oa, va, xa + st * kEBox + 16 * u);
                if (lb && (hb >> 28)) rewalk(eb0, ob, vb, xb + st * kEBox + 16 * u);
            }
        }
        __syncwarp();   // every lane consumed the buffer before it is refilled
        if (lane == 0 && st + kEStages < nst) {
            mbar_expect_tx(mbar0 + 8 * slot, kEStage);
            tma_load_2d(buf, &tmap, (int32_t)((st + kEStages) * kEBox), (int32_t)row0, mbar0 + 8 * slot);
        }
        if (++slot == kEStages) {
            slot = 0;
            phase ^= 1u;
        }
    }
    // the remainder past the last full row belongs to the last chunk (reading C7)
    if (la && ta == P.p - 1) {
        uint32_t s = (ea & 0xFFFFu) >> 11;
        for (uint64_t a = (ta + 1) * P.L; a < P.n; ++a) step1(s, oa, P.in[a], a);
    }
    if (lb && tb == P.p - 1) {
        uint32_t s = (eb & 0xFFFFu) >> 11;
        for (uint64_t a = (tb + 1) * P.L; a < P.n; ++a) step1(s, ob, P.in[a], a);
    }
}

// symbol-major lanes tables (entry = dest * ES | acc << (8 ES - 1)): shared memory when the
// table fits (SMEM), else global / L2
template <bool W32, bool SMEM>
__global__ void __launch_bounds__(kFindThreads) find_emit_lanes_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    constexpr uint32_t ES = W32 ? 4 : 2, ACC = W32 ? 31 : 15;
    const uint32_t COL = d.Qpad * ES, SMASK = (d.Qpad - 1u) * ES, CMASK = d.Apad - 1u;
    const unsigned char* g = reinterpret_cast<const unsigned char*>(d.lanes_tab);
    uint32_t sbase = 0;
    if (SMEM) {   // staged at a multiple of the column stride: the base ORs into offsets
        const uint32_t sraw = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        sbase = (sraw + COL - 1) / COL * COL;
        const size_t bytes = (size_t)d.Apad * COL;
        const uint4* src = reinterpret_cast<const uint4*>(d.lanes_tab);
        uint4* dst = reinterpret_cast<uint4*>(sm + (sbase - sraw));
        for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.p) return;
    const uint64_t b0 = find_b(P, t), b1 = find_b(P, t + 1);
    uint32_t e = P.fchunk_q[t] * ES;
    unsigned long long o = P.fchunk_base[t];
    auto look = [&](uint32_t c) {
        const uint32_t off = (e & SMASK) | ((c & CMASK) * COL + sbase);
        if constexpr (SMEM) {
            if constexpr (W32) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(off));
            else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(e) : "r"(off));
        } else {
            e = W32 ? __ldg(reinterpret_cast<const uint32_t*>(g + off))
                    : __ldg(reinterpret_cast<const uint16_t*>(g + off));
        }
    };
    auto step = [&](uint32_t c, uint64_t k) {   // predicated store, no branch
        look(c);
        const uint32_t h = e >> ACC;
        if (h && o < P.fmax) P.fout[o] = k;
        o += h;
    };
    uint64_t a = b0;
    for (; a < b1 && (((uintptr_t)(P.in + a)) & 15u); ++a) step(P.in[a], a);
    uint4 nx = a + 16 <= b1 ? ldg_v4_na(P.in + a) : make_uint4(0, 0, 0, 0);
    for (; a + 16 <= b1; a += 16) {
        const uint4 x = nx;
        if (a + 32 <= b1) nx = ldg_v4_na(P.in + a + 16);
        const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) step(__byte_perm(w4[q], 0u, 0x4440u | k), a + 4 * q + k);
    }
    for (; a < b1; ++a) step(P.in[a], a);
}

// ---- route trace (parem_trace_async): the visited states of every chunk that meets the
// window [tlo, thi), walked from the chunk's true entering state (Alg. 1's Rr of the route the
// join selects).  One generic kernel for both table classes (global tables). ----
__global__ void __launch_bounds__(kFindThreads) find_trace_kernel(const MatchParams P) {
    const DevDfa& d = P.d;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.p) return;
    const uint64_t b0 = find_b(P, t), b1 = find_b(P, t + 1);
    if (b1 <= P.tlo || b0 >= P.thi) return;
    const uint64_t end = min(b1, P.thi);
    const uint32_t A = d.A, Qpad = d.Qpad;
    const bool tiny = d.lanes_tab == nullptr;
    uint32_t s = P.fchunk_q[t];
    auto step = [&](uint32_t c, uint64_t k) {
        c = c < A ? c : A - 1u;   // ESYMBOL inputs: any in-table column (the trace is unspecified)
        if (tiny) s = __ldg(d.tab1 + s * A + c) & 0x7FFFu;
        else if (d.lanes_u32) s = (__ldg(reinterpret_cast<const uint32_t*>(d.lanes_tab) + (size_t)c * Qpad + s) & ((Qpad - 1u) * 4u)) >> 2;
        else s = (__ldg(reinterpret_cast<const uint16_t*>(d.lanes_tab) + (size_t)c * Qpad + s) & ((Qpad - 1u) * 2u)) >> 1;
        if (k >= P.tlo) P.tout[k - P.tlo] = (d.has_sink && s == d.sink) ? PAREM_DEAD : s;
    };
    uint64_t a = b0;
    for (; a < end && (((uintptr_t)(P.in + a)) & 15u); ++a) step(P.in[a], a);
    for (; a + 16 <= end; a += 16) {
        const uint4 x = ldg_v4_na(P.in + a);
        const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) step(__byte_perm(w4[q], 0u, 0x4440u | k), a + 4 * q + k);
    }
    for (; a < end; ++a) step(P.in[a], a);
}

unsigned nblk(uint64_t n, uint32_t per) { return (unsigned)((n + per - 1) / per); }

}  // namespace

// Workspace after the match's own: q, h per chunk; u64 bases; scan block sums; tiny path:
// per-chunk maps (end u8, hits u32) and per-group maps.
size_t find_extra_bytes(const Plan& plan, const DevDfa& d) {
    const uint64_t p = plan.p, groups = (p + kGroup - 1) / kGroup, nb = (p + kScanBlock - 1) / kScanBlock;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t s = al(4 * p) + al(4 * p) + al(8 * p) + al(8 * nb) + al(4 * groups);
    const uint64_t nsg = (groups + 31) / 32;
    if (plan.kernel == kKernelTiny)
        s += al((size_t)p * d.Qpad) + al(4 * (size_t)p * d.Qpad) + al(4 * (size_t)groups * d.Qpad) +
             al(8 * (size_t)groups * d.Qpad) + al(4 * (size_t)nsg * d.Qpad) + al(4 * nsg);
    return s;
}

void find_bind(const Plan& plan, MatchParams& P, unsigned char* extra) {
    const uint64_t p = plan.p, groups = (p + kGroup - 1) / kGroup, nb = (p + kScanBlock - 1) / kScanBlock;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    unsigned char* o = extra;
    P.fchunk_q = reinterpret_cast<uint32_t*>(o); o += al(4 * p);
    P.fchunk_h = reinterpret_cast<uint32_t*>(o); o += al(4 * p);
    P.fchunk_base = reinterpret_cast<unsigned long long*>(o); o += al(8 * p);
    P.fblock = reinterpret_cast<unsigned long long*>(o); o += al(8 * nb);
    P.fgq = reinterpret_cast<uint32_t*>(o); o += al(4 * groups);
    if (plan.kernel == kKernelTiny) {
        P.fmend = o; o += al((size_t)p * P.d.Qpad);
        P.fmhits = reinterpret_cast<uint32_t*>(o); o += al(4 * (size_t)p * P.d.Qpad);
        P.fgend = reinterpret_cast<uint32_t*>(o); o += al(4 * (size_t)groups * P.d.Qpad);
        P.fghits = reinterpret_cast<unsigned long long*>(o); o += al(8 * (size_t)groups * P.d.Qpad);
        const uint64_t nsg = (groups + 31) / 32;
        P.fsend = reinterpret_cast<uint32_t*>(o); o += al(4 * (size_t)nsg * P.d.Qpad);
        P.fsq = reinterpret_cast<uint32_t*>(o); o += al(4 * nsg);
    }
}

int launch_find(const Plan& plan, const MatchParams& P, cudaStream_t s) {
    const uint64_t p = plan.p, groups = (p + kGroup - 1) / kGroup, nb = (p + kScanBlock - 1) / kScanBlock;
    if (plan.kernel == kKernelTiny) {
        find_group_kernel<<<nblk(groups * 32, kFindThreads), kFindThreads, 0, s>>>(P, groups);
        prof_after("find_group", s);
        const uint64_t nsg = (groups + 31) / 32;
        find_super_kernel<<<nblk(nsg * 32, kFindThreads), kFindThreads, 0, s>>>(P, groups);
        prof_after("find_super", s);
        find_group_seq_kernel<<<1, 32, 0, s>>>(P, groups);
        prof_after("find_group_seq", s);
        find_group_in_kernel<<<nblk(nsg * 32, kFindThreads), kFindThreads, 0, s>>>(P, groups);
        prof_after("find_group_in", s);
        find_chunks_kernel<<<nblk(groups, kFindThreads), kFindThreads, 0, s>>>(P, groups);
        prof_after("find_resolve", s);
    } else if (plan.kernel == kKernelLanes) {
        find_lanes_seq_kernel<<<1, 32, 0, s>>>(P);
        prof_after("find_resolve", s);
    }   // converging path: q_i and h_i were written by conv_resolve
    if (P.tout) {   // route trace instead of match positions
        if (P.thi > P.tlo) find_trace_kernel<<<nblk(p, kFindThreads), kFindThreads, 0, s>>>(P);
        prof_after("find_trace", s);
        const cudaError_t te = cudaGetLastError();
        if (te != cudaSuccess) {
            set_error("trace kernel: %s", cudaGetErrorString(te));
            return PAREM_ECUDA;
        }
        return PAREM_OK;
    }
    find_scan_sums_kernel<<<(unsigned)nb, kScanBlock / 4, 0, s>>>(P);
    prof_after("find_scan_sums", s);
    find_scan_blocks_kernel<<<1, 32, 0, s>>>(P, nb);
    prof_after("find_scan_blocks", s);
    find_scan_apply_kernel<<<(unsigned)nb, kScanBlock / 4, 0, s>>>(P);
    prof_after("find_scan", s);
    CUtensorMap emap;
    const bool etma = plan.kernel == kKernelTiny && P.d.sym_bits && plan.policy == PAREM_BOUNDARY_GRID &&
                      !(((uintptr_t)P.in) & 15u) && P.L % kEBox == 0 && P.L >= kEBox && P.p * P.L <= P.n &&
                      emit_tma_smem(P.d) <= 232448 && encode_rows_map(&emap, P.in, P.L, P.p, kEBox, kERows);
    if (etma) {
        const size_t smem = emit_tma_smem(P.d);
        const void* fn = P.d.sym_bits == 2 ? (const void*)find_emit_stride_tma_kernel<2>
                                           : (const void*)find_emit_stride_tma_kernel<1>;
        smem_optin(fn, smem);
        void* args[] = {const_cast<MatchParams*>(&P), &emap};
        cudaLaunchKernel(fn, dim3(nblk(p, kEThreads * 2)), dim3(kEThreads), args, smem, s);
    } else if (plan.kernel == kKernelTiny && P.d.sym_bits) {
        const size_t smem = (size_t)P.d.Qp * 2048 + (size_t)P.d.Qp * P.d.A * 2;
        const void* fn = P.d.sym_bits == 2 ? (const void*)find_emit_stride_kernel<2> : (const void*)find_emit_stride_kernel<1>;
        smem_optin(fn, smem);
        void* args[] = {const_cast<MatchParams*>(&P)};
        cudaLaunchKernel(fn, dim3(nblk(p, kFindThreads)), dim3(kFindThreads), args, smem, s);
    } else if (plan.kernel == kKernelTiny) {
        const size_t smem = (size_t)P.d.Qp * P.d.A * 2;
        find_emit_tiny_kernel<<<nblk(p, kFindThreads), kFindThreads, smem, s>>>(P);
    } else {
        const size_t ES = P.d.lanes_u32 ? 4 : 2, tb = (size_t)P.d.Apad * P.d.Qpad * ES;
        const bool smem = tb <= (size_t)160 * 1024;
        const size_t sm = smem ? tb + (size_t)P.d.Qpad * ES : 0;   // + alignment slack
        const void* fn = P.d.lanes_u32 ? (smem ? (const void*)find_emit_lanes_kernel<true, true>
                                               : (const void*)find_emit_lanes_kernel<true, false>)
                                       : (smem ? (const void*)find_emit_lanes_kernel<false, true>
                                               : (const void*)find_emit_lanes_kernel<false, false>);
        if (smem) smem_optin(fn, sm);
        void* args[] = {const_cast<MatchParams*>(&P)};
        cudaLaunchKernel(fn, dim3(nblk(p, kFindThreads)), dim3(kFindThreads), args, sm, s);
    }
    prof_after("find_emit", s);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("find kernels: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    return PAREM_OK;
}

}  // namespace parem
