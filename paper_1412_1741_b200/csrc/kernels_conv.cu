// kernels_conv.cu -- the CONVERGING multi-start path for large DFAs (internal states > 32,
// complete tables): PaREM's candidate sets R_i are walked with
// in-flight route merging: routes of one chunk that reach the
// same state follow the same path for the rest of the chunk (Table II shows it: P_2's
// routes from 0 and 7 meet after two symbols), so each chunk costs
// sum_t |delta*(R_i, T[b_i, b_i + t))| lookups instead of |R_i| * len_i.  Results are the
// sequential ones exactly: the per-chunk map start -> (end, hits) is never approximated,
// it is evaluated at the one start state the join needs.
//
// Launches per match (all graph-capturable):
//   K1 conv_set     warp per chunk: walk the SET R_i (deduplicated each step) until at most
//                   dmax distinct states remain at offset m_i (hand-over); if the chunk ends
//                   first, its <= 32 phase-B states are the survivors, walked to the end
//                   ("open"); a set that never shrank to 32 states is "wide";
//   K2 conv_follow  thread per chunk: walk the <= 4 handed-over survivors z_k over the rest
//                   of the chunk -> (end_k, tail hits_k);
//   E1..E5          the join as a composition of small maps: each chunk's end set (<= 32
//                   states, 1 once its routes merged), each chunk as a map from the previous
//                   end set (head walks, lanes of a warp), block composition, one warp along
//                   q0's path, per-chunk resolution and the result.  Wide chunks are
//                   resolved by one warp in chunk order (whole-chunk walks from their
//                   entering set), the rest in parallel.
// Every input byte is validated once (reading C11): K2 tails, E2 heads and open tails.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>

#include <mutex>
#include <type_traits>

#include "kernels_common.cuh"

namespace parem {

namespace {

constexpr uint32_t kDMax = 4;             // survivors handed from K1 to K2
constexpr uint32_t kSetWarps = 8;         // K1: warps (= chunks) per CTA
constexpr uint32_t kFollowThreads = 512;  // K2 / K3: threads (= chunks) per CTA

struct ConvChunk {      // 64 B per chunk in the workspace
    uint32_t m;         // bytes covered by the set walk (the head)
    uint32_t D;         // survivors handed over (1..kDMax); 0 = open (head = whole chunk)
    uint32_t z[kDMax];  // survivor states at b_i + m (padded with z[0])
    uint32_t end[kDMax];
    uint32_t tail[kDMax];
    uint32_t anchor;    // K2: every survivor ended in one state
    uint32_t q;         // J: true state at b_i
};
static_assert(sizeof(ConvChunk) == 64, "ConvChunk");

// Survivors of a chunk once its set walk has shrunk to <= 32 states: z[k] at offset m (the
// head), walked to the chunk end -> end[k], tail hits tail[k]; eidx[k] = index of end[k] in
// the chunk's end set.  Every chunk has one (n = 0 only for a "wide" chunk whose set never
// shrank to 32 states).
constexpr uint32_t kMaxSurv = 32;
constexpr uint32_t kWide = 0xFFFFFFFFu;
// WsHeader::err bits of the converging path
constexpr uint32_t kErrUnsound = 1u;   // a state entered a chunk that its candidate set does not hold: EINTERNAL
constexpr uint32_t kErrWide = 4u;      // some chunk is wide (conv_wide_kernel has work)
struct SurvRec {
    uint32_t n;
    uint32_t z[kMaxSurv];
    uint32_t end[kMaxSurv];
    uint32_t tail[kMaxSurv];
    uint8_t eidx[kMaxSurv];
    uint32_t pad;
};
struct EndSet {        // distinct end states of a chunk (the possible entering states of the next)
    uint32_t n;
    uint32_t s[kMaxSurv];
    uint32_t pad;
};
struct MapRec {        // chunk i as a map over the end set of chunk i-1 (entering index j)
    uint8_t idx[kMaxSurv];     // -> index into this chunk's end set
    uint32_t hits[kMaxSurv];   // hits of the walk through this chunk
};
constexpr uint32_t kBlk = 32;   // chunks per composed block
struct BlockMap {
    uint8_t idx[kMaxSurv];
};

struct ConvWs {        // the converging path's workspace after the 256-byte header area
    ConvChunk* info;
    SurvRec* surv;
    EndSet* ends;
    MapRec* maps;
    BlockMap* bmaps;   // per block of kBlk chunks
    BlockMap* smaps;   // per super-block of kBlk blocks
    uint32_t* bin;     // entering index per block
    uint32_t* sin;     // entering index per super-block
};

__host__ __device__ __forceinline__ size_t alw(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ __forceinline__ size_t conv_ws_bytes(uint64_t p) {
    const uint64_t nb = (p + kBlk - 1) / kBlk;
    const uint64_t ns = (nb + kBlk - 1) / kBlk;
    return alw(p * sizeof(ConvChunk)) + alw(p * sizeof(SurvRec)) + alw(p * sizeof(EndSet)) +
           alw(p * sizeof(MapRec)) + alw(nb * sizeof(BlockMap)) + alw(ns * sizeof(BlockMap)) + alw(4 * (nb + 1)) +
           alw(4 * (ns + 1));
}

__device__ __forceinline__ ConvWs conv_ws(const MatchParams& P) {
    const uint64_t p = P.p, nb = (p + kBlk - 1) / kBlk;
    unsigned char* o = reinterpret_cast<unsigned char*>(P.maps);
    ConvWs w;
    w.info = reinterpret_cast<ConvChunk*>(o); o += alw(p * sizeof(ConvChunk));
    w.surv = reinterpret_cast<SurvRec*>(o); o += alw(p * sizeof(SurvRec));
    w.ends = reinterpret_cast<EndSet*>(o); o += alw(p * sizeof(EndSet));
    w.maps = reinterpret_cast<MapRec*>(o); o += alw(p * sizeof(MapRec));
    const uint64_t ns = (nb + kBlk - 1) / kBlk;
    w.bmaps = reinterpret_cast<BlockMap*>(o); o += alw(nb * sizeof(BlockMap));
    w.smaps = reinterpret_cast<BlockMap*>(o); o += alw(ns * sizeof(BlockMap));
    w.bin = reinterpret_cast<uint32_t*>(o); o += alw(4 * (nb + 1));
    w.sin = reinterpret_cast<uint32_t*>(o);
    return w;
}

__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

// K1 per-warp scratch: the candidate list (u16 state indices, compacted in place) and, for
// Qpad <= 256, the owner tags (u16 per state: the list index that last produced the
// state), else a Qpad-bit image bitmap (atomicOr; the tags would cost the occupancy).
constexpr int kPark = 4;   // parked chunks per warp in the set walk's phase B
constexpr uint32_t kOwnerMaxQ = 256;   // measured: tags win on cfg3 (256 states), lose on cfg5 (1024)
__host__ __device__ __forceinline__ size_t set_warp_bytes(uint32_t cap, uint32_t Qpad) {
    return al16(2 * (size_t)cap) + (Qpad <= kOwnerMaxQ ? al16(2 * (size_t)Qpad) : al16((size_t)(Qpad + 31) / 32 * 4));
}

__host__ __device__ __forceinline__ size_t tab_bytes(const DevDfa& d) {
    return (size_t)d.Apad * d.Qpad * (d.lanes_u32 ? 4 : 2);
}

// Symbol-major table access (entry = dest * ES | acc << (8 ES - 1)): the next entry of a
// route at entry e under symbol c is at byte offset (e & SMASK) | col(c).
template <bool SMEM, bool W32>
struct Tab {
    static constexpr uint32_t ES = W32 ? 4 : 2, ACC = W32 ? 31 : 15;
    static constexpr bool kSmem = SMEM, kW32 = W32, kRep = false, kHyb = false, kByte = false;
    const unsigned char* g;
    uint32_t cbase, COL, SMASK, CMASK;

    __device__ __forceinline__ void init(const DevDfa& d, uint32_t sbase) {
        g = reinterpret_cast<const unsigned char*>(d.lanes_tab);
        COL = d.Qpad * ES;
        SMASK = (d.Qpad - 1u) * ES;
        CMASK = d.Apad - 1u;   // keeps invalid bytes (ESYMBOL) inside the table
        cbase = SMEM ? sbase : 0u;
    }
    __device__ __forceinline__ uint32_t col(uint32_t c) const { return (c & CMASK) * COL + cbase; }
    // column of an input byte already masked to (c & CMASK) by a whole-word AND
    __device__ __forceinline__ uint32_t colm(uint32_t c) const { return c * COL + cbase; }
    __device__ __forceinline__ uint32_t at(uint32_t off) const {
        uint32_t v;
        if constexpr (SMEM) {
            if constexpr (W32) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(off));
            else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(off));
        } else {
            using ET = typename std::conditional<W32, uint32_t, uint16_t>::type;
            v = __ldg(reinterpret_cast<const ET*>(g + off));
        }
        return v;
    }
    __device__ __forceinline__ uint32_t next(uint32_t e, uint32_t colc) const { return at((e & SMASK) | colc); }
    __device__ __forceinline__ uint32_t state(uint32_t e) const { return (e & SMASK) / ES; }
    __device__ __forceinline__ uint32_t hit(uint32_t e) const { return e >> ACC; }
    __device__ __forceinline__ uint32_t start(uint32_t s) const { return s * ES; }
    __device__ __forceinline__ uint32_t word_mask() const { return CMASK * 0x01010101u; }
};

// Stage the symbol-major table into shared memory at an address that is a multiple of its
// column stride (so the shared base ORs into column offsets); returns that address.
template <bool SMEM, bool W32>
__device__ __forceinline__ uint32_t stage_table(const DevDfa& d, unsigned char* sm) {
    if (!SMEM) return 0u;
    constexpr uint32_t ES = W32 ? 4 : 2;
    const uint32_t COL = d.Qpad * ES;
    const uint32_t sraw = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t sbase = (sraw + COL - 1) / COL * COL;
    const size_t bytes = tab_bytes(d);
    const uint4* src = reinterpret_cast<const uint4*>(d.lanes_tab);
    uint4* dst = reinterpret_cast<uint4*>(sm + (sbase - sraw));
    for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    return sbase;
}

__host__ __device__ __forceinline__ size_t smem_tab_bytes(const DevDfa& d, bool smem) {
    return smem ? al16(tab_bytes(d) + (size_t)d.Qpad * (d.lanes_u32 ? 4 : 2)) : 0;
}

// Replicated-fragment table for the follow walk (shared memory, R = 8, 16 or 32 copies of
// a u16 table): 32 lanes looking up 32 random states of a plain table hit ~3.5 wavefronts
// per LDS (profiles/r01_ncu_full_cfg3_follow*).  Copy k = lane mod R lives in the banks
// k + R j (j < 32 / R), so only the 32 / R lanes sharing a copy can conflict, and every
// entry stores the NEXT state's address fragment within its copy (+ accept bit 15):
// next = (e & FMASK) | col(c), one LOP3 per lookup as with the plain table.
//   frag(s, k) = (s >> 1 >> lg) << 7 | ((s >> 1) & (32/R - 1)) * R * 4 | k << 2 | (s & 1) << 1,
//   lg = log2(32 / R); a column (one symbol) is Qpad * 2 R bytes.
template <int R>
__host__ __device__ __forceinline__ uint32_t rep_frag(uint32_t s, uint32_t k) {
    constexpr uint32_t G = 32 / R, LG = R == 32 ? 0 : R == 16 ? 1 : 2;
    const uint32_t w = s >> 1;
    return ((w >> LG) << 7) | ((w & (G - 1u)) * (R * 4u)) | (k << 2) | ((s & 1u) << 1);
}
__host__ __device__ __forceinline__ uint32_t rep_col_bytes(uint32_t Qpad, uint32_t R) { return Qpad * 2u * R; }

template <int R>
struct TabR {
    static constexpr uint32_t ES = 2;
    static constexpr bool kSmem = true, kW32 = false, kRep = true, kHyb = false, kByte = false;
    static constexpr int kR = R;
    uint32_t tbase, COL, FMASK, AM1, k;

    // stage the copies into shared memory at tbase (a multiple of COL) inside [sm, sm + bytes)
    __device__ __forceinline__ void init(const DevDfa& d, unsigned char* sm) {
        COL = rep_col_bytes(d.Qpad, R);
        FMASK = COL - 1u;
        AM1 = d.A - 1u;
        k = threadIdx.x & (uint32_t)(R - 1);
        const uint32_t sraw = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        tbase = (sraw + COL - 1) / COL * COL;
        unsigned char* base = sm + (tbase - sraw);
        const uint32_t total = d.A * d.Qpad;   // one thread per (c, s) entry writes its R copies
        for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
            const uint32_t s = i & (d.Qpad - 1u), c = i >> d.log2Qpad;
            uint32_t dest, acc;
            if (d.lanes_u32) {
                const uint32_t e = __ldg(reinterpret_cast<const uint32_t*>(d.lanes_tab) + (size_t)c * d.Qpad + s);
                dest = (e & ((d.Qpad - 1u) * 4u)) >> 2;
                acc = e >> 31;
            } else {
                const uint32_t e = __ldg(reinterpret_cast<const uint16_t*>(d.lanes_tab) + (size_t)c * d.Qpad + s);
                dest = (e & ((d.Qpad - 1u) * 2u)) >> 1;
                acc = e >> 15;
            }
            unsigned char* colp = base + (size_t)c * COL;
#pragma unroll 4
            for (uint32_t kk = 0; kk < (uint32_t)R; ++kk)
                *reinterpret_cast<uint16_t*>(colp + rep_frag<R>(s, kk)) = (uint16_t)(rep_frag<R>(dest, kk) | (acc << 15));
        }
    }
    // bytes >= A use column A - 1 (the chunk reports ESYMBOL anyway, reading C11)
    __device__ __forceinline__ uint32_t col(uint32_t c) const { return min(c, AM1) * COL + tbase; }
    __device__ __forceinline__ uint32_t colm(uint32_t c) const { return min(c, AM1) * COL + tbase; }
    __device__ __forceinline__ uint32_t next(uint32_t e, uint32_t colc) const {
        uint32_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"((e & FMASK) | colc));
        return v;
    }
    __device__ __forceinline__ uint32_t state(uint32_t e) const {
        constexpr uint32_t G = 32 / R, LG = R == 32 ? 0 : R == 16 ? 1 : 2;
        const uint32_t f = e & FMASK;
        const uint32_t w = ((f >> 7) << LG) | ((f >> 2) / R & (G - 1u));
        return (w << 1) | ((f >> 1) & 1u);
    }
    __device__ __forceinline__ uint32_t hit(uint32_t e) const { return e >> 15; }
    __device__ __forceinline__ uint32_t start(uint32_t s) const { return rep_frag<R>(s, k); }
    __device__ __forceinline__ uint32_t word_mask() const { return 0xFFFFFFFFu; }
};

__host__ __device__ __forceinline__ size_t rep_smem_bytes(const DevDfa& d, uint32_t R) {
    const size_t col = rep_col_bytes(d.Qpad, R);
    return col > (1u << 15) ? 0 : (size_t)d.A * col + col;   // + alignment slack
}

// Byte-entry replicated table for the follow walk of DFAs with <= 256 states: sixteen copies of
// a u8 table in shared memory, copy k = lane mod 16 in banks {2k, 2k+1} (eight states per
// 128-byte row and copy), so only the two lanes that share a copy can conflict: 2 wavefronts
// per lookup instead of the ~3.6 of 32 random lanes in one plain table -- what bounds the cfg3
// follow (profiles/r02_ncu_full_cfg3_conv_follow.json).  With one byte per entry the 16 copies
// of a 256 x 26 table take 104 KB (u16 entries: 208 KB, which starves the input streams'
// L1).  A byte holds the state only, so states are renumbered inside the kernel -- accepting
// states last -- and the accept flag is the comparison code >= Qpad - |F|.
struct TabB {
    static constexpr bool kSmem = true, kW32 = false, kRep = false, kHyb = false, kByte = true;
    static constexpr uint32_t kBudget = 112u * 1024u;
    uint32_t tbase, COL, AM1, k8, hitK, lgQ, cof, sof;

    __host__ __device__ static uint32_t col_bytes(const DevDfa& d) { return d.Qpad * 16u; }
    __host__ __device__ static bool applies(const DevDfa& d) {
        return d.Qpad <= 256u && !d.has_sink && (size_t)d.A * col_bytes(d) <= kBudget;
    }
    __host__ __device__ static size_t bytes(const DevDfa& d) {
        return (size_t)d.A * col_bytes(d) + col_bytes(d) + 512u;   // + alignment slack + the two code maps
    }
    __device__ __forceinline__ void init(const DevDfa& d, unsigned char* sm) {
        COL = col_bytes(d);
        AM1 = d.A - 1u;
        k8 = (threadIdx.x & 15u) * 8u;
        const uint32_t sraw = smem_u32(sm);
        tbase = (sraw + COL - 1) / COL * COL;
        unsigned char* base = sm + (tbase - sraw);
        unsigned char* code_of = base + (size_t)d.A * COL;   // state -> code
        unsigned char* state_of = code_of + 256;             // code -> state
        cof = smem_u32(code_of);
        sof = smem_u32(state_of);
        // codes: non-accepting states first (in state order), accepting states last
        uint32_t nacc = 0;
        for (uint32_t t = 0; t < d.Qp; ++t) nacc += d.acc[t];
        hitK = 256u - d.Qpad + nacc;   // code >= Qpad - nacc  <=>  code + hitK carries out of 8 bits
        lgQ = d.log2Qpad;
        for (uint32_t s = threadIdx.x; s < d.Qpad; s += blockDim.x) {
            uint32_t code = s;
            if (s < d.Qp) {
                uint32_t before_same = 0;
                const uint32_t a = d.acc[s];
                for (uint32_t t = 0; t < s; ++t) before_same += (d.acc[t] == a);
                code = a ? d.Qpad - nacc + before_same : before_same;
            } else {
                code = s - nacc;   // unused padding states fill the gap below the accepting codes
            }
            code_of[s] = (unsigned char)code;
            state_of[code] = (unsigned char)s;
        }
        __syncthreads();
        const uint32_t total = d.A * d.Qpad;
        for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
            const uint32_t s = i & (d.Qpad - 1u), c = i >> d.log2Qpad;
            uint32_t dest;
            if (d.lanes_u32) dest = (__ldg(reinterpret_cast<const uint32_t*>(d.lanes_tab) + (size_t)c * d.Qpad + s) & ((d.Qpad - 1u) * 4u)) >> 2;
            else dest = (__ldg(reinterpret_cast<const uint16_t*>(d.lanes_tab) + (size_t)c * d.Qpad + s) & ((d.Qpad - 1u) * 2u)) >> 1;
            const uint32_t cs = code_of[s], cd = code_of[dest];
            unsigned char* row = base + (size_t)c * COL + (cs >> 3) * 128u + (cs & 7u);
#pragma unroll 4
            for (uint32_t kk = 0; kk < 16u; ++kk) row[kk * 8u] = (unsigned char)cd;
        }
    }
    __device__ __forceinline__ uint32_t col(uint32_t c) const { return min(c, AM1) * COL + (tbase | k8); }
    __device__ __forceinline__ uint32_t colm(uint32_t c) const { return min(c, AM1) * COL + (tbase | k8); }
    // e = code (8 bits)
    __device__ __forceinline__ uint32_t next(uint32_t e, uint32_t colc) const {
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(colc | ((e & 0xF8u) << 4) | (e & 7u)));
        return v;
    }
    __device__ __forceinline__ uint32_t state(uint32_t e) const {
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(sof + e));
        return v;
    }
    __device__ __forceinline__ uint32_t hit(uint32_t e) const { return (e + hitK) >> 8; }
    __device__ __forceinline__ uint32_t start(uint32_t s) const {
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(cof + s));
        return v;
    }
    __device__ __forceinline__ uint32_t word_mask() const { return 0xFFFFFFFFu; }
};

// Hybrid table for the follow walk of tables that do not fit shared memory (cfg5: 1024 x 256,
// 512 KiB): the first CS symbol columns live in shared memory, PACKED three 10-bit states per
// word (WPC = ceil(Qpad / 3) words per column), the other columns are read from the u16 table
// in global memory (L1/L2).  The selection is branch-free: a lane served from shared memory
// aims its global load at entry 0 (one shared wavefront for all such lanes), a lane served
// from global memory aims its shared load at word 0 (a broadcast); ptxas turns a per-lane
// LDS/LDG choice into a divergent branch, which was 2x slower (profiles/r02_conv_sweeps.txt,
// g25).  Accept flags come from a Qpad-bit bitmap in shared memory (the packed entries have
// no room for them).  The L2 gather rate bounds the all-global walk (~1.1 lookups/clk/SM,
// tools/follow_probe.cu); with 144 of 256 columns in shared memory and two chunks per
// thread the probe reaches 1.7 (profiles/r02_follow_probe.txt).
struct TabH {
    static constexpr bool kSmem = true, kW32 = false, kRep = false, kHyb = true, kByte = false;
    static constexpr uint32_t kBudget = 192u * 1024u;   // more starves the L1 the input stream needs
    const uint16_t* g;
    uint32_t sbase, abase, CS, WPC, Qpad, AM1, CMASK;

    __host__ __device__ static uint32_t wpc(uint32_t Qpad) { return (Qpad + 2u) / 3u; }
    __host__ __device__ static uint32_t columns(const DevDfa& d) {
        const uint32_t c = (kBudget - d.Qpad / 8u - 32u) / (wpc(d.Qpad) * 4u);
        return c < d.A ? c : d.A;
    }
    __host__ __device__ static bool applies(const DevDfa& d) {
        // u16 table, 10-bit states, and enough columns on chip to matter
        return !d.lanes_u32 && d.Qpad <= 1024u && 5u * columns(d) >= 2u * d.A;
    }
    __host__ __device__ static size_t bytes(const DevDfa& d) {
        return (size_t)columns(d) * wpc(d.Qpad) * 4u + d.Qpad / 8u + 32u;
    }
    __device__ __forceinline__ void init(const DevDfa& d, unsigned char* sm) {
        g = reinterpret_cast<const uint16_t*>(d.lanes_tab);
        CS = columns(d);
        WPC = wpc(d.Qpad);
        Qpad = d.Qpad;
        AM1 = d.A - 1u;
        CMASK = d.Apad - 1u;
        uint32_t* pw = reinterpret_cast<uint32_t*>(sm);
        sbase = smem_u32(pw);
        for (uint32_t i = threadIdx.x; i < CS * WPC; i += blockDim.x) {
            const uint32_t c = i / WPC, q = i - c * WPC;
            uint32_t w = 0;
#pragma unroll
            for (uint32_t r = 0; r < 3; ++r) {
                const uint32_t st = 3u * q + r;
                if (st < Qpad) w |= (((uint32_t)__ldg(g + (size_t)c * Qpad + st) & 0x7FFFu) >> 1) << (10u * r);
            }
            pw[i] = w;
        }
        uint32_t* aw = pw + CS * WPC;
        abase = smem_u32(aw);
        for (uint32_t i = threadIdx.x; i < (Qpad + 31u) / 32u; i += blockDim.x) {
            uint32_t w = 0;
            for (uint32_t b = 0; b < 32u; ++b) {
                const uint32_t st = 32u * i + b;
                if (st < d.Qp && d.acc[st]) w |= 1u << b;
            }
            aw[i] = w;
        }
    }
    __device__ __forceinline__ uint32_t col(uint32_t c) const { return min(c, AM1); }
    __device__ __forceinline__ uint32_t colm(uint32_t c) const { return c; }   // c <= CMASK < Apad
    // e = state | accept << 31
    __device__ __forceinline__ uint32_t next(uint32_t e, uint32_t c) const {
        const uint32_t st = e & 0x3FFu;
        const bool insm = c < CS;
        const uint32_t q = (st * 43691u) >> 17, r = st - 3u * q;
        const uint32_t vg = __ldg(g + (insm ? 0u : c * Qpad + st));
        uint32_t ww, aw;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ww) : "r"(sbase + 4u * (insm ? c * WPC + q : 0u)));
        const uint32_t dst = insm ? (ww >> (r * 10u)) & 0x3FFu : (vg & 0x7FFu) >> 1;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(aw) : "r"(abase + ((dst >> 5) << 2)));
        return dst | (((aw >> (dst & 31u)) & 1u) << 31);
    }
    // the same lookup for a route that may be switched off: a dead route aims both loads at
    // the dummy addresses (no extra wavefronts) and its result is ignored by the caller --
    // keeps the multi-route walk free of branches
    __device__ __forceinline__ uint32_t next_live(uint32_t e, uint32_t c, bool live) const {
        const uint32_t st = e & 0x3FFu;
        const bool insm = c < CS;
        const uint32_t q = (st * 43691u) >> 17, r = st - 3u * q;
        const uint32_t vg = __ldg(g + ((live && !insm) ? c * Qpad + st : 0u));
        uint32_t ww, aw;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ww) : "r"(sbase + 4u * ((live && insm) ? c * WPC + q : 0u)));
        const uint32_t dst = insm ? (ww >> (r * 10u)) & 0x3FFu : (vg & 0x7FFu) >> 1;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(aw) : "r"(abase + ((dst >> 5) << 2)));
        return dst | (((aw >> (dst & 31u)) & 1u) << 31);
    }
    __device__ __forceinline__ uint32_t state(uint32_t e) const { return e & 0x3FFu; }
    __device__ __forceinline__ uint32_t hit(uint32_t e) const { return e >> 31; }
    __device__ __forceinline__ uint32_t start(uint32_t s) const { return s; }
    __device__ __forceinline__ uint32_t word_mask() const { return CMASK * 0x01010101u; }
};

// staging and footprint of any follow table type
template <class TT>
__device__ __forceinline__ void tab_setup(TT& T, const DevDfa& d, unsigned char* sm) {
    if constexpr (TT::kRep || TT::kHyb || TT::kByte) T.init(d, sm);
    else T.init(d, stage_table<TT::kSmem, TT::kW32>(d, sm));
}
template <class TT>
__host__ __device__ __forceinline__ size_t tab_smem(const DevDfa& d) {
    if constexpr (TT::kHyb || TT::kByte) return TT::bytes(d);
    else if constexpr (TT::kRep) return rep_smem_bytes(d, TT::kR);
    else return smem_tab_bytes(d, TT::kSmem);
}

__device__ __forceinline__ uint64_t conv_b(const MatchParams& P, uint64_t i) {
    return i >= P.p ? P.n : i * P.L;   // GRID boundaries (reading C7)
}

// ---------------------------------------------------------------------------------------
// K1: set walk.  Persistent warps take chunks in turn; R_t is deduplicated every step
// (phase A) until <= 32 states remain.  For Qpad <= 256 each element writes its list
// index into the owner tag of the state it reaches (plain shared stores, last writer
// wins), and after a warp barrier exactly one element per distinct state reads its own
// index back -- no atomics, no bitmap to clear; larger Q uses an image bitmap and atomicOr.
// The chunk is then PARKED in one of kPark register slots (one state per lane) and the
// warp advances its parked chunks together, 32 bytes at a time (kPark independent lookup
// chains per lane), counting distinct states with __match_any_sync after every 32 bytes.
// A chunk leaves phase B when <= dmax states remain (hand-over) or at its end (open).
template <bool SMEM, bool W32, bool OWN>
__global__ void __launch_bounds__(kSetWarps * 32) conv_set_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t cap = P.slots;   // max |R_i|
    const size_t tb = smem_tab_bytes(d, SMEM);
    Tab<SMEM, W32> T;
    T.init(d, stage_table<SMEM, W32>(d, sm));
    __syncthreads();
    unsigned char* ws = sm + tb + warp * set_warp_bytes(cap, d.Qpad);
    uint16_t* list = reinterpret_cast<uint16_t*>(ws);   // state indices, compacted in place
    uint16_t* owner = reinterpret_cast<uint16_t*>(ws + al16(2 * (size_t)cap));
    uint32_t* bm = reinterpret_cast<uint32_t*>(owner);
    const uint32_t nbm = (d.Qpad + 31) / 32;
    const uint8_t* in = P.in;
    const uint32_t ltmask = (1u << lane) - 1u;
    const uint32_t dmax = P.dmax;
    const ConvWs W = conv_ws(P);
    ConvChunk* infos = W.info;

    // distinct states among the warp's lanes (lanes past |R| duplicate lane 0)
    auto distinct = [&](uint32_t e, uint32_t& leaders) {
        const uint32_t m = __match_any_sync(0xFFFFFFFFu, e & T.SMASK);
        leaders = __ballot_sync(0xFFFFFFFFu, (__ffs(m) - 1) == (int)lane);
        return (uint32_t)__popc(leaders);
    };
    // a chunk whose set never shrank to 32 states: no survivors (resolved in order later)
    auto write_wide = [&](uint64_t t, uint64_t b0, uint64_t b1) {
        if (lane == 0) {
            infos[t].m = (uint32_t)(b1 - b0);
            infos[t].D = kWide;
            W.surv[t].n = 0;
        }
    };
    // open chunk (routes did not merge to <= dmax by its end): the survivors are its <= 32
    // distinct END states and its head is the whole chunk (the join walks it from each
    // possible entering state)
    auto write_open = [&](uint64_t t, uint64_t b0, uint64_t b1, uint32_t e, uint32_t leaders, uint32_t nd) {
        SurvRec& s = W.surv[t];
        if ((leaders >> lane) & 1u) {
            const uint32_t r = __popc(leaders & ltmask);
            s.z[r] = T.state(e);
            s.end[r] = T.state(e);
            s.tail[r] = 0;
        }
        if (lane == 0) {
            s.n = nd;
            infos[t].m = (uint32_t)(b1 - b0);
            infos[t].D = 0;
        }
    };
    // survivors z_0 .. z_{nd-1}: the leader lanes in lane order, padded with z_0
    auto write_handover = [&](uint64_t t, uint64_t m, uint32_t e, uint32_t leaders, uint32_t nd) {
        const uint32_t s = T.state(e);
        const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, s, __ffs(leaders) - 1);
        if ((leaders >> lane) & 1u) infos[t].z[__popc(leaders & ltmask)] = s;
        if (lane >= nd && lane < kDMax) infos[t].z[lane] = s0;
        if (lane == 0) {
            infos[t].m = (uint32_t)m;
            infos[t].D = nd;
        }
    };

    uint64_t pt[kPark], ppos[kPark], pb0[kPark], pb1[kPark];
    uint32_t pe[kPark];
    uint32_t occ = 0;   // occupied slots (warp-uniform)
    unsigned long long lk = 0;   // lookups at distinct states (warp-uniform; hdr->lookups)
    uint64_t tn = (uint64_t)blockIdx.x * kSetWarps + warp;
    const uint64_t tstride = (uint64_t)gridDim.x * kSetWarps;
    for (;;) {
        // ---- refill free slots: A2 + phase A of the next chunks ----
        while (occ != (1u << kPark) - 1u && tn < P.p) {
            const uint64_t t = tn;
            tn += tstride;
            const uint64_t b0 = conv_b(P, t), b1 = conv_b(P, t + 1);
            // A2: R_t = L(T[b_t - 1]) (complete tables: S = Q), R_0 = {q0}
            uint32_t D;
            __syncwarp();
            if (t == 0) {
                bool dead;
                D = 1;
                if (lane == 0) list[0] = (uint16_t)start_state(P, &dead);
            } else {
                const uint32_t c = in[b0 - 1];
                if (c >= d.A && P.cand != PAREM_CANDIDATES_ENUM) {
                    // invalid byte (the result is ESYMBOL, reading C11): any candidate will
                    // do, and all of Q would not fit the list sized for max |L(c)|
                    D = 1;
                    if (lane == 0) list[0] = 0;
                } else {
                    const uint32_t li = P.cand == PAREM_CANDIDATES_ENUM ? d.A : c;
                    D = __ldg(d.Lcnt + li);
                    const uint32_t* L = d.Llist + __ldg(d.Loff + li);
                    for (uint32_t k = lane; k < D; k += 32) list[k] = (uint16_t)__ldg(L + k);
                }
            }
            __syncwarp();
            uint64_t pos = b0;
            // phase A: more than 32 states -- the deduplicated image every step
            while (D > 32 && pos < b1) {
                const uint32_t colc = T.col(__ldg(in + pos));
                uint32_t nD = 0;
                lk += D;
                if constexpr (OWN) {
                    // pass 1: image of every element, in place; owner tag of its state
                    for (uint32_t base = 0; base < D; base += 128) {
                        uint32_t ns[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t i = base + 32u * j + lane;
                            ns[j] = i < D ? T.state(T.next(list[i] * T.ES, colc)) : 0u;
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t i = base + 32u * j + lane;
                            if (i < D) {
                                list[i] = (uint16_t)ns[j];
                                owner[ns[j]] = (uint16_t)i;
                            }
                        }
                    }
                    __syncwarp();
                    // pass 2: the element that owns its state survives; compaction in place
                    for (uint32_t base = 0; base < D; base += 32) {
                        const uint32_t i = base + lane;
                        const uint32_t v = i < D ? list[i] : 0u;
                        const bool fresh = i < D && owner[v] == (uint16_t)i;
                        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, fresh);
                        if (fresh) list[nD + __popc(bal & ltmask)] = (uint16_t)v;
                        nD += __popc(bal);
                    }
                } else {
                    // large Q: image bitmap, atomicOr decides the first arrival (a batch is
                    // read into registers before any of its writes land)
                    for (uint32_t i = lane; i < nbm; i += 32) bm[i] = 0u;
                    __syncwarp();
                    for (uint32_t base = 0; base < D; base += 128) {
                        uint32_t ns[4];
                        bool fresh[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t idx = base + 32u * j + lane;
                            ns[j] = idx < D ? T.state(T.next(list[idx] * T.ES, colc)) : 0xFFFFFFFFu;
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            fresh[j] = false;
                            if (ns[j] != 0xFFFFFFFFu) {
                                const uint32_t bit = 1u << (ns[j] & 31u);
                                fresh[j] = !(atomicOr(bm + (ns[j] >> 5), bit) & bit);
                            }
                        }
                        __syncwarp();
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, fresh[j]);
                            if (fresh[j]) list[nD + __popc(bal & ltmask)] = (uint16_t)ns[j];
                            nD += __popc(bal);
                        }
                        __syncwarp();
                    }
                }
                if constexpr (OWN) __syncwarp();
                D = nD;
                ++pos;
            }
            if (D > 32) {   // reached the chunk end in phase A
                write_wide(t, b0, b1);
                continue;
            }
            const uint32_t e = (lane < D ? list[lane] : list[0]) * T.ES;
            uint32_t leaders;
            const uint32_t nd = distinct(e, leaders);
            if (nd <= dmax) {
                write_handover(t, pos - b0, e, leaders, nd);
                continue;
            }
            if (pos >= b1) {
                write_open(t, b0, b1, e, leaders, nd);
                continue;
            }
            const int k = __ffs(~occ) - 1;   // park it
#pragma unroll
            for (int j = 0; j < kPark; ++j)
                if (j == k) {
                    pt[j] = t;
                    ppos[j] = pos;
                    pb0[j] = b0;
                    pb1[j] = b1;
                    pe[j] = e;
                }
            occ |= 1u << k;
        }
        if (!occ) break;
        // ---- phase B: advance every parked chunk by up to 32 bytes, chains interleaved
        // (lanes whose routes met keep walking in lock-step: the same address costs no
        // extra L1TEX wavefront) ----
        uint32_t cnt[kPark], mine[kPark], cmax = 0;
#pragma unroll
        for (int j = 0; j < kPark; ++j) {
            cnt[j] = ((occ >> j) & 1u) ? (uint32_t)min((uint64_t)32, pb1[j] - ppos[j]) : 0u;
            mine[j] = lane < cnt[j] ? (uint32_t)__ldg(in + ppos[j] + lane) : 0u;
            cmax = max(cmax, cnt[j]);
        }
        for (uint32_t i = 0; i < cmax; ++i) {
#pragma unroll
            for (int j = 0; j < kPark; ++j) {
                const uint32_t c = __shfl_sync(0xFFFFFFFFu, mine[j], i);
                if (i < cnt[j]) pe[j] = T.next(pe[j], T.col(c));
            }
        }
#pragma unroll
        for (int j = 0; j < kPark; ++j) {
            if (!((occ >> j) & 1u)) continue;
            ppos[j] += cnt[j];
            uint32_t leaders;
            const uint32_t nd = distinct(pe[j], leaders);
            lk += (unsigned long long)cnt[j] * nd;   // >= nd distinct states during these bytes
            if (nd <= dmax) {
                write_handover(pt[j], ppos[j] - pb0[j], pe[j], leaders, nd);
                occ &= ~(1u << j);
            } else if (ppos[j] >= pb1[j]) {
                write_open(pt[j], pb0[j], pb1[j], pe[j], leaders, nd);
                occ &= ~(1u << j);
            }
        }
    }
    if (lane == 0 && lk) atomicAdd(&P.hdr->lookups, lk);
}

// ---------------------------------------------------------------------------------------
// K2: follow the survivors over the rest of the chunk, thread per chunk (CPT chunks per
// thread, interleaved: CPT independent chains), K routes per chunk in registers with K =
// the warp's largest survivor count (4, or 1); routes k >= D of a chunk are predicated
// off.  Once every lane of the warp has all its routes in one state (warp-uniform), one
// route is advanced and the others rebuilt exactly (end shared, hits + the offset at the
// merge point).
template <class TT, int CPT>
struct Follow {
    const TT& T;
    const uint8_t* p[CPT];
    uint32_t nv[CPT], D[CPT];
    uint32_t e[CPT][kDMax], h[CPT][kDMax];
    uint32_t bad, A, wmask, K, K7F;   // K = (256 - A) per byte, K7F = K & 0x7F7F7F7F
    bool check;
    // Per-lane merging (NEXT-2 (ii)): slots [0, Dl) of chunk j hold the routes still walked.
    // Every check merges routes that are in the same state PAIRWISE: the higher slot k is
    // retired into the lower slot r -- the last live slot moves into slot k, and the freed
    // slot Dl - 1 keeps the record of the retired route (survivor id, its carrier's survivor
    // id, its hit offset against the carrier at the meeting point).  The hot loop's
    // predicate stays "k < Dl"; predicated-off lookups issue no L1TEX wavefronts, which is
    // what bounds the walk (the slowest lane of the warp no longer makes every lane pay
    // kDMax lookups per byte).  sid = slot -> survivor id (2 bits each).  finish() rebuilds
    // every survivor's (end, hits) in survivor order.
    uint32_t Dl[CPT], sid[CPT];
    uint32_t mv[CPT];   // sum over retired routes of the 16-byte vectors they walked (stats)

    __device__ __forceinline__ Follow(const TT& t) : T(t) {}

    __device__ __forceinline__ void begin(int j) {
        Dl[j] = D[j];
        sid[j] = 0xE4u;   // slot k holds survivor k
        mv[j] = 0;
    }
    // retire slot K into slot R (R < K < Dl), written for compile-time K, R, LAST = Dl - 1
    template <int R, int K, int LAST>
    __device__ __forceinline__ void retire(int j) {
        const uint32_t off = h[j][K] - h[j][R];   // u32 wrap-around is exact
        const uint32_t idk = (sid[j] >> (2 * K)) & 3u, idr = (sid[j] >> (2 * R)) & 3u, idl = (sid[j] >> (2 * LAST)) & 3u;
        if (K != LAST) {
            e[j][K] = e[j][LAST];
            h[j][K] = h[j][LAST];
        }
        e[j][LAST] = idr;   // record of the retired route, kept in the freed slot
        h[j][LAST] = off;
        uint32_t sd = sid[j] & ~((3u << (2 * K)) | (3u << (2 * LAST)));
        sd |= idl << (2 * K);      // (K == LAST: overwritten by the next line)
        sd = (sd & ~(3u << (2 * LAST))) | (idk << (2 * LAST));
        sid[j] = sd;
    }
    // true when chunk j walks one route (now or already)
    __device__ __forceinline__ bool lane_merge(int j, uint32_t vdone) {
        static_assert(kDMax == 4, "lane_merge / finish are written out for 4 routes");
        // at most Dl - 1 retirements; each pass retires the first equal pair it finds
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
            const uint32_t n = Dl[j];
            if (n <= 1u) break;
            const uint32_t s0 = T.state(e[j][0]), s1 = T.state(e[j][1]), s2 = T.state(e[j][2]), s3 = T.state(e[j][3]);
            bool did = true;
            if (n == 2u) {
                if (s1 == s0) retire<0, 1, 1>(j);
                else did = false;
            } else if (n == 3u) {
                if (s1 == s0) retire<0, 1, 2>(j);
                else if (s2 == s0) retire<0, 2, 2>(j);
                else if (s2 == s1) retire<1, 2, 2>(j);
                else did = false;
            } else {
                if (s1 == s0) retire<0, 1, 3>(j);
                else if (s2 == s0) retire<0, 2, 3>(j);
                else if (s3 == s0) retire<0, 3, 3>(j);
                else if (s2 == s1) retire<1, 2, 3>(j);
                else if (s3 == s1) retire<1, 3, 3>(j);
                else if (s3 == s2) retire<2, 3, 3>(j);
                else did = false;
            }
            if (!did) break;
            Dl[j] = n - 1u;
            mv[j] += vdone;
        }
        return Dl[j] <= 1u;
    }
    // One 32-bit word of EVERY chunk of the thread, byte by byte with the chunks interleaved
    // (b -> j -> k): the CPT chains of a thread overlap their lookups (issue is in order, so
    // walking chunk 0's sixteen bytes before chunk 1's would serialise them).  Hybrid tables
    // use the switched lookup (no branch per route); on[j] = chunk j has this vector.
    template <int K>
    __device__ __forceinline__ void words(const uint32_t (&w)[CPT], const bool (&on)[CPT]) {
        uint32_t wm[CPT];
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            if (check && on[j]) {
                const uint32_t t = (w[j] & 0x7F7F7F7Fu) + K7F;
                bad |= (w[j] & this->K) | ((w[j] | this->K) & t);
            }
            wm[j] = w[j] & wmask;
        }
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) {
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const uint32_t colc = T.colm(__byte_perm(wm[j], 0u, 0x4440u | b));
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const bool live = on[j] && (K == 1 || (uint32_t)k < Dl[j]);
                    if constexpr (TT::kHyb) {
                        const uint32_t ne = T.next_live(e[j][k], colc, live);
                        e[j][k] = live ? ne : e[j][k];
                        h[j][k] += live ? T.hit(ne) : 0u;
                    } else {
                        if (live) {
                            e[j][k] = T.next(e[j][k], colc);
                            h[j][k] += T.hit(e[j][k]);
                        }
                    }
                }
            }
        }
    }

    // lookups of chunk j over `bytes` bytes, `head` of them before the 16-byte vectors:
    // routes still live walked every byte, a retired route walked up to its meeting point
    __device__ __forceinline__ unsigned long long chunk_lookups(int j, uint64_t bytes, uint64_t head) const {
        if (D[j] <= 1u) return bytes;
        const uint64_t nret = D[j] - Dl[j];
        return bytes * Dl[j] + min(bytes * nret, head * nret + (uint64_t)16 * mv[j]);
    }
    // rebuild every survivor's (entry, hits): live slots first, then the retired records from
    // the LAST retirement to the first (slots Dl .. D - 1 ascending), so that a carrier --
    // live, or retired later than its rider -- is final before the rider reads it
    __device__ __forceinline__ void finish() {
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            if (D[j] <= 1u || Dl[j] == D[j]) continue;
            uint32_t fe[kDMax], fh[kDMax];
#pragma unroll
            for (int k = 0; k < (int)kDMax; ++k) fe[k] = fh[k] = 0;
#pragma unroll
            for (int sl = 0; sl < (int)kDMax; ++sl) {
                if ((uint32_t)sl >= D[j]) continue;
                const uint32_t id = (sid[j] >> (2 * sl)) & 3u;
                uint32_t ve, vh;
                if ((uint32_t)sl < Dl[j]) {
                    ve = e[j][sl];
                    vh = h[j][sl];
                } else {
                    const uint32_t c = e[j][sl] & 3u;   // carrier's survivor id
                    ve = c == 0u ? fe[0] : c == 1u ? fe[1] : c == 2u ? fe[2] : fe[3];
                    vh = (c == 0u ? fh[0] : c == 1u ? fh[1] : c == 2u ? fh[2] : fh[3]) + h[j][sl];
                }
#pragma unroll
                for (int k = 0; k < (int)kDMax; ++k)
                    if (id == (uint32_t)k) {
                        fe[k] = ve;
                        fh[k] = vh;
                    }
            }
#pragma unroll
            for (int k = 0; k < (int)kDMax; ++k) {
                e[j][k] = fe[k];
                h[j][k] = fh[k];
            }
            Dl[j] = D[j];
            sid[j] = 0xE4u;
        }
    }

    template <int K>
    __device__ __forceinline__ void word(int j, uint32_t w) {
        if (check) {
            // bytes >= A (reading C11): b >= A iff b + (256 - A) carries out of bit 7 = the
            // majority of (b7, K7, carry into bit 7); accumulated, tested once at the end
            const uint32_t t = (w & 0x7F7F7F7Fu) + K7F;
            bad |= (w & K) | ((w | K) & t);
        }
        const uint32_t wm = w & wmask;
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) {
            const uint32_t colc = T.colm(__byte_perm(wm, 0u, 0x4440u | b));
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (K == 1 || (uint32_t)k < Dl[j]) {
                    e[j][k] = T.next(e[j][k], colc);
                    h[j][k] += T.hit(e[j][k]);
                }
            }
        }
    }

    // Walk the 16-byte vectors of every chunk (warp-uniform bound nvmax) with PF vectors
    // per chain in flight (a register ring: a thread-per-chunk stream needs ~64 B in flight
    // per chain to cover HBM latency behind the dependent lookups; one vector was not
    // enough, tools/gather_probe.cu rep16).  Routes run K = kDMax wide until every lane of
    // the warp has all routes of all its chunks in one state (warp-uniform, checked every 4
    // vectors), then one route per chunk; the others are rebuilt at the end (rebuild()).
    static constexpr int PF = CPT == 1 ? 4 : 2;
    bool merged;

    __device__ __forceinline__ void run(uint32_t nvmax, bool multi) {
        merged = !multi;
        uint4 ring[CPT][PF];
#pragma unroll
        for (int j = 0; j < CPT; ++j)
#pragma unroll
            for (int u = 0; u < PF; ++u)
                ring[j][u] = (uint32_t)u < nv[j] ? ldg_v4_na(p[j] + 16ull * u) : make_uint4(0, 0, 0, 0);
        for (uint32_t v = 0; v < nvmax; v += PF) {
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const uint32_t vv = v + u;
                uint4 x[CPT];
#pragma unroll
                for (int j = 0; j < CPT; ++j) {
                    x[j] = ring[j][u];
                    if (vv + PF < nv[j]) ring[j][u] = ldg_v4_na(p[j] + 16ull * (vv + PF));
                }
                if constexpr (CPT > 1 || TT::kHyb) {
                    bool on[CPT];
                    uint32_t w0[CPT], w1[CPT], w2[CPT], w3[CPT];
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        on[j] = vv < nv[j];
                        w0[j] = x[j].x;
                        w1[j] = x[j].y;
                        w2[j] = x[j].z;
                        w3[j] = x[j].w;
                    }
                    if (merged) {
                        words<1>(w0, on);
                        words<1>(w1, on);
                        words<1>(w2, on);
                        words<1>(w3, on);
                    } else {
                        words<kDMax>(w0, on);
                        words<kDMax>(w1, on);
                        words<kDMax>(w2, on);
                        words<kDMax>(w3, on);
                    }
                } else if (merged) {
#pragma unroll
                    for (int j = 0; j < CPT; ++j)
                        if (vv < nv[j]) {
                            word<1>(j, x[j].x);
                            word<1>(j, x[j].y);
                            word<1>(j, x[j].z);
                            word<1>(j, x[j].w);
                        }
                } else {
#pragma unroll
                    for (int j = 0; j < CPT; ++j)
                        if (vv < nv[j]) {
                            word<kDMax>(j, x[j].x);
                            word<kDMax>(j, x[j].y);
                            word<kDMax>(j, x[j].z);
                            word<kDMax>(j, x[j].w);
                        }
                }
                if (!merged) {
                    if ((vv & 3u) == 3u) {
                        bool conv = true;
#pragma unroll
                        for (int j = 0; j < CPT; ++j) conv &= lane_merge(j, vv + 1u);
                        if (__all_sync(0xFFFFFFFFu, conv)) merged = true;
                    }
                }
            }
        }
    }

    __device__ __forceinline__ void step1(int j, uint32_t c) {
        if (check && c >= A) bad |= 0x80u;
        const uint32_t colc = T.col(c);
#pragma unroll
        for (int k = 0; k < (int)kDMax; ++k)
            if ((uint32_t)k < Dl[j]) {
                e[j][k] = T.next(e[j][k], colc);
                h[j][k] += T.hit(e[j][k]);
            }
    }
};

template <class TT, int CPT>
__global__ void __launch_bounds__(kFollowThreads, 1) conv_follow_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    TT T;
    tab_setup(T, d, sm);
    __syncthreads();
    const ConvWs W = conv_ws(P);
    const uint8_t* in = P.in;
    Follow<TT, CPT> F(T);
    F.bad = 0;
    F.A = d.A;
    F.check = d.A < 256;
    F.K = ((256u - d.A) & 0xFFu) * 0x01010101u;
    F.K7F = F.K & 0x7F7F7F7Fu;
    F.wmask = T.word_mask();
    uint64_t t[CPT], a[CPT], b1[CPT], a0[CPT], hdb[CPT];
    bool act[CPT];
    const uint64_t tb = (uint64_t)blockIdx.x * blockDim.x * CPT + threadIdx.x;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        t[j] = tb + (uint64_t)j * blockDim.x;
        const bool live = t[j] < P.p;
        const ConvChunk* info = W.info + (live ? t[j] : 0);
        const uint64_t b0 = conv_b(P, t[j]);
        b1[j] = live ? conv_b(P, t[j] + 1) : b0;
        const uint32_t D0 = live ? info->D : 0u;
        F.D[j] = D0 == kWide ? 0u : D0;   // follow only handed-over chunks
        F.begin(j);
        act[j] = F.D[j] != 0;
        a[j] = act[j] ? b0 + info->m : b1[j];
#pragma unroll
        for (int k = 0; k < (int)kDMax; ++k) {
            F.e[j][k] = act[j] ? T.start(info->z[k]) : 0u;
            F.h[j][k] = 0;
        }
        // unaligned head (< 16 bytes)
        const uint64_t mis = act[j] ? (uint64_t)(((uintptr_t)(in + a[j])) & 15u) : 0u;
        uint64_t hd = mis ? a[j] + (16 - mis) : a[j];
        if (hd > b1[j]) hd = b1[j];
        a0[j] = a[j];
        hdb[j] = hd - a[j];
        for (; a[j] < hd; ++a[j]) F.step1(j, in[a[j]]);
        F.nv[j] = act[j] ? (uint32_t)((b1[j] - a[j]) >> 4) : 0u;
        F.p[j] = in + a[j];
    }
    // 16-byte vectors: a warp-uniform trip count (lanes past their own end idle) and a
    // warp-uniform route count
    uint32_t nvmax = 0, Dw = 0;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        nvmax = max(nvmax, F.nv[j]);
        Dw = max(Dw, F.D[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nvmax = max(nvmax, __shfl_xor_sync(0xFFFFFFFFu, nvmax, o));
        Dw = max(Dw, __shfl_xor_sync(0xFFFFFFFFu, Dw, o));
    }
    F.run(nvmax, Dw > 1);
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        a[j] += (uint64_t)F.nv[j] << 4;
        for (; act[j] && a[j] < b1[j]; ++a[j]) F.step1(j, in[a[j]]);
    }
    {
        unsigned long long lk = 0;
#pragma unroll
        for (int j = 0; j < CPT; ++j)
            if (act[j]) lk += F.chunk_lookups(j, b1[j] - a0[j], hdb[j]);
        lk = warp_sum(lk);
        if ((threadIdx.x & 31u) == 0 && lk) atomicAdd(&P.hdr->lookups, lk);
    }
    F.finish();
    const bool anybad = (F.bad & 0x80808080u) != 0;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        if (!act[j]) continue;
        SurvRec& sr = W.surv[t[j]];
        const ConvChunk* info = W.info + t[j];
        sr.n = F.D[j];
#pragma unroll
        for (int k = 0; k < (int)kDMax; ++k)
            if ((uint32_t)k < F.D[j]) {
                sr.z[k] = info->z[k];
                sr.end[k] = T.state(F.e[j][k]);
                sr.tail[k] = F.h[j][k];
            }
        if (anybad) {
            const uint64_t off = first_bad(in, conv_b(P, t[j]) + info->m, b1[j], d.A);
            if (off < b1[j]) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
        }
    }
}

// K2 with TMA-staged input (the default): chunk t is row t of a 2-D tensor view of the
// input (row length L); each warp owns 32 consecutive chunks and streams them through
// shared memory in 32-row x 64-byte boxes (cp.async.bulk.tensor.2d, SWIZZLE_64B, two
// mbarrier stages), so the input costs one TMA transaction per 2 KB instead of 32 L1TEX
// wavefronts per 16-byte vector load of a thread-per-chunk stream (the follow walk was
// L1TEX-bound: profiles/r02_ncu_*follow*).  A lane walks its head remainder (from b_t + m_t
// to the next 16-byte unit) from global memory, then its staged units; the last chunk
// (not a full row) is walked from global memory.
constexpr uint32_t kFBox = 64, kFStages = 2, kFStageBytes = 32 * kFBox, kFThreads = 512;

__host__ __device__ __forceinline__ size_t follow_tma_smem(size_t tb) {
    return ((tb + 1023) & ~(size_t)1023) + (kFThreads / 32) * (kFStages * kFStageBytes + 8 * kFStages) + 1024;
}

// COOP = true replaces the TMA engine by warp-cooperative cp.async copies on the LSU path
// (lane l copies 16-byte unit l & 3 of rows 8 i + (l >> 2), i = 0..3, into the same 64B-swizzled
// stage layout): a stream of 32-row x 64-byte boxes is bound by the TMA engine's per-row rate
// (profiles/r02_conv_sweeps.txt), while four cp.async instructions touch 8 lines each.
template <class TT, bool COOP>
__global__ void __launch_bounds__(kFThreads, 1) conv_follow_tma_kernel(const MatchParams P,
                                                                    const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char sm[];
    const DevDfa& d = P.d;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    TT T;
    tab_setup(T, d, sm);
    const size_t tb = tab_smem<TT>(d);
    const uint32_t sraw = smem_u32(sm);
    const uint32_t stg = (sraw + (uint32_t)tb + 1023u) & ~1023u;   // 1024-aligned staging (swizzle atoms)
    const uint32_t stage0 = stg + warp * kFStages * kFStageBytes;
    const uint32_t mbar0 = stg + nw * kFStages * kFStageBytes + warp * kFStages * 8u;
    const ConvWs W = conv_ws(P);
    const uint8_t* in = P.in;
    const uint64_t pfull = P.p - 1;   // rows covered by the tensor map (the last chunk is not a full row)
    const uint32_t nst = (uint32_t)(P.L / kFBox);
    const uint64_t row0 = (uint64_t)blockIdx.x * blockDim.x + warp * 32u;
    const uint64_t t = row0 + lane;

    Follow<TT, 1> F(T);
    F.bad = 0;
    F.A = d.A;
    F.check = d.A < 256;
    F.wmask = T.word_mask();
    F.K = ((256u - d.A) & 0xFFu) * 0x01010101u;
    F.K7F = F.K & 0x7F7F7F7Fu;
    const bool live = t < P.p;
    const ConvChunk* info = W.info + (live ? t : 0);
    const uint64_t b0 = conv_b(P, t), b1 = live ? conv_b(P, t + 1) : b0;
    const uint32_t D0 = live ? info->D : 0u;
    F.D[0] = D0 == kWide ? 0u : D0;   // follow only handed-over chunks
    F.begin(0);
    const bool act = F.D[0] != 0;
    const uint32_t m = act ? info->m : 0u;
#pragma unroll
    for (int k = 0; k < (int)kDMax; ++k) {
        F.e[0][k] = act ? T.start(info->z[k]) : 0u;
        F.h[0][k] = 0;
    }
    const bool staged = act && t < pfull;
    // first staged 16-byte unit of this row; bytes [m, 16 su) are walked from global memory
    const uint32_t su = staged ? (m + 15u) >> 4 : 0xFFFFFFFFu;
    uint32_t s_lo = su >> 2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s_lo = min(s_lo, __shfl_xor_sync(0xFFFFFFFFu, s_lo, o));
    const bool warp_staged = s_lo < nst;
    // cooperative copy of box sb of this warp's 32 rows into stage buffer `buf` (one commit group)
    auto coop_issue = [&](uint32_t sb, uint32_t buf) {
        if (sb < nst) {
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
                const uint32_t r = 8u * i + (lane >> 2), u = lane & 3u;
                if (row0 + r < pfull) {
                    const uint8_t* src = in + (row0 + r) * P.L + (uint64_t)sb * kFBox + 16u * u;
                    const uint32_t dst = buf + r * kFBox + ((u ^ ((r >> 1) & 3u)) << 4);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if constexpr (COOP) {
        if (warp_staged)
            for (uint32_t k = 0; k < kFStages; ++k) coop_issue(s_lo + k, stage0 + k * kFStageBytes);
    } else if (lane == 0 && warp_staged) {
        for (uint32_t k = 0; k < kFStages; ++k) mbar_init(mbar0 + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t k = 0; k < kFStages && s_lo + k < nst; ++k) {
            mbar_expect_tx(mbar0 + 8 * k, kFStageBytes);
            tma_load_2d(stage0 + k * kFStageBytes, &tmap, (int32_t)((s_lo + k) * kFBox), (int32_t)row0, mbar0 + 8 * k);
        }
    }
    __syncthreads();   // table staged, barriers initialised

    if (staged) {
        const uint64_t hb = b0 + min((uint64_t)su * 16u, b1 - b0);
        for (uint64_t a = b0 + m; a < hb; ++a) F.step1(0, in[a]);
    }
    const uint32_t Dw = __reduce_max_sync(0xFFFFFFFFu, staged ? F.D[0] : 0u);
    bool merged = Dw <= 1;
    if (warp_staged) {
        const uint32_t sw = (lane >> 1) & 3u, off = lane * kFBox;
        uint32_t slot = 0, phase = 0;
        for (uint32_t s = s_lo; s < nst; ++s) {
            if constexpr (COOP) {
                // the oldest group (this slot's) is complete for this lane's copies; the warp
                // barrier makes every lane's copies visible
                asm volatile("cp.async.wait_group %0;" ::"n"(kFStages - 1) : "memory");
                __syncwarp();
            } else {
                mbar_wait(mbar0 + 8 * slot, phase);
            }
            const uint32_t buf = stage0 + slot * kFStageBytes;
            uint4 x[4];
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) x[u] = lds128(buf + off + ((u ^ sw) << 4));
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                if (4 * s + u < su) continue;   // before this row's first staged unit (or not staged)
                if (merged) {
                    F.template word<1>(0, x[u].x);
                    F.template word<1>(0, x[u].y);
                    F.template word<1>(0, x[u].z);
                    F.template word<1>(0, x[u].w);
                } else {
                    F.template word<kDMax>(0, x[u].x);
                    F.template word<kDMax>(0, x[u].y);
                    F.template word<kDMax>(0, x[u].z);
                    F.template word<kDMax>(0, x[u].w);
                }
            }
            // refill this slot only after every lane consumed its staged words (the TMA
            // write must not overtake an in-flight shared load of the same buffer)
            __syncwarp();
            if constexpr (COOP) {
                coop_issue(s + kFStages, buf);   // always commits, so the group count stays in step
            } else if (lane == 0 && s + kFStages < nst) {
                mbar_expect_tx(mbar0 + 8 * slot, kFStageBytes);
                tma_load_2d(buf, &tmap, (int32_t)((s + kFStages) * kFBox), (int32_t)row0, mbar0 + 8 * slot);
            }
            if (++slot == kFStages) {
                slot = 0;
                phase ^= 1u;
            }
            if (!merged) {
                const bool conv = !staged || F.lane_merge(0, 4u * (s + 1u) > su ? 4u * (s + 1u) - su : 0u);
                if (__all_sync(0xFFFFFFFFu, conv)) merged = true;
            }
        }
    }
    {
        // The last chunk is not a full row: its lane walks it with the thread-stream loop
        // (16-byte vectors, prefetch ring).  A byte-at-a-time walk of up to L bytes by ONE
        // thread took longer than the whole staged part (3 ms for a 56 KB chunk) and was
        // what made every staged variant look slow until round 2's last session.
        const bool lastc = act && !staged;
        uint64_t a = b0 + m;
        if (lastc) {
            const uint64_t mis = (uint64_t)(((uintptr_t)(in + a)) & 15u);
            uint64_t hd = mis ? a + (16 - mis) : a;
            if (hd > b1) hd = b1;
            for (; a < hd; ++a) F.step1(0, in[a]);
        }
        F.nv[0] = lastc ? (uint32_t)((b1 - a) >> 4) : 0u;
        F.p[0] = in + a;
        const uint32_t nvl = __reduce_max_sync(0xFFFFFFFFu, F.nv[0]);
        if (nvl) F.run(nvl, true);   // warp-uniform call; lanes without vectors idle
        if (lastc)
            for (a += (uint64_t)F.nv[0] << 4; a < b1; ++a) F.step1(0, in[a]);
    }
    {
        // staged rows: head = bytes up to the first staged 16-byte unit
        const uint64_t bytes = act ? b1 - (b0 + m) : 0u;
        unsigned long long lk = act ? F.chunk_lookups(0, bytes, staged ? min((uint64_t)su * 16u - (uint64_t)m, bytes) : bytes) : 0u;
        lk = warp_sum(lk);
        if (lane == 0 && lk) atomicAdd(&P.hdr->lookups, lk);
    }
    F.finish();
    if (!act) return;
    SurvRec& sr = W.surv[t];
    sr.n = F.D[0];
#pragma unroll
    for (int k = 0; k < (int)kDMax; ++k)
        if ((uint32_t)k < F.D[0]) {
            sr.z[k] = info->z[k];
            sr.end[k] = T.state(F.e[0][k]);
            sr.tail[k] = F.h[0][k];
        }
    if (F.bad & 0x80808080u) {
        const uint64_t off = first_bad(in, b0 + m, b1, d.A);
        if (off < b1) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
    }
}

// Walk one route from state q over in[a, b) (global table, any alignment); hits optional.
template <bool W32>
__device__ __forceinline__ uint32_t walk1(const DevDfa& d, const uint8_t* in, uint64_t a, uint64_t b, uint32_t q,
                                          uint32_t* hits) {
    Tab<false, W32> T;
    T.init(d, 0u);
    uint32_t e = q * T.ES, h = 0;
    for (; a < b && (((uintptr_t)(in + a)) & 15u); ++a) {
        e = T.next(e, T.col(in[a]));
        h += T.hit(e);
    }
    uint4 nx = a + 16 <= b ? ldg_v4_na(in + a) : make_uint4(0, 0, 0, 0);
    for (; a + 16 <= b; a += 16) {
        const uint4 x = nx;
        if (a + 32 <= b) nx = ldg_v4_na(in + a + 16);
        const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2)
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                e = T.next(e, T.col(__byte_perm(w4[q2], 0u, 0x4440u | k)));
                h += T.hit(e);
            }
    }
    for (; a < b; ++a) {
        e = T.next(e, T.col(in[a]));
        h += T.hit(e);
    }
    if (hits) *hits = h;
    return T.state(e);
}

// ---------------------------------------------------------------------------------------
// The join, as a composition of SMALL maps.  Chunk i's possible entering
// states are the end set of chunk i-1 (<= 32 states; 1 when its routes merged).  E2 walks
// each of them over chunk i's head [b_i, b_i + m_i) (lanes of one warp, same bytes),
// matches the state reached against chunk i's survivors and so turns chunk i into a map
// "entering index -> (end-set index, hits)".  E3 composes blocks of 32 such maps (lane =
// entering index), E4 walks the block maps along q0's path, E5 resolves every chunk's
// entering state and hits in parallel and writes the result.  Every step is parallel
// whether or not routes merged; only "wide" chunks (the set never shrank to 32 states)
// are resolved by one warp in chunk order (conv_wide_kernel), each from its entering set.

// E1: end set of every chunk (distinct survivor ends) and each survivor's index in it.
__global__ void __launch_bounds__(kFollowThreads) conv_ends_kernel(const MatchParams P) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.p) return;
    const ConvWs W = conv_ws(P);
    SurvRec& s = W.surv[t];
    EndSet& es = W.ends[t];
    if (W.info[t].D == kWide) {   // resolved by conv_wide_kernel from its entering set
        es.n = 0;
        atomicOr(&P.hdr->err, kErrWide);
        return;
    }
    uint32_t n = 0;
    for (uint32_t k = 0; k < s.n; ++k) {
        const uint32_t v = s.end[k];
        uint32_t j = 0;
        while (j < n && es.s[j] != v) ++j;
        if (j == n) es.s[n++] = v;
        s.eidx[k] = (uint8_t)j;
    }
    es.n = n;
}

// E1b: "wide" chunks (their set walk never shrank to 32 states), in chunk order, by one
// warp: lane j walks the WHOLE chunk from state j of the previous chunk's end set (<= 32;
// a wide predecessor was resolved just before), the distinct end states become this
// chunk's end set and its map is written directly.  Runs only if a wide chunk exists;
// every other chunk stays on the parallel path.
template <bool W32>
__global__ void conv_wide_kernel(const MatchParams P) {
    if (threadIdx.x >= 32 || !(P.hdr->err & kErrWide)) return;
    const uint32_t lane = threadIdx.x;
    const ConvWs W = conv_ws(P);
    const DevDfa& d = P.d;
    Tab<false, W32> T;
    T.init(d, 0u);
    const uint8_t* in = P.in;
    unsigned long long routes = 0, steps = 0;
    for (uint64_t t0 = 0; t0 < P.p; t0 += 32) {
        const bool w = t0 + lane < P.p && W.info[t0 + lane].D == kWide;
        uint32_t wide = __ballot_sync(0xFFFFFFFFu, w);
        while (wide) {
            const uint64_t t = t0 + (uint64_t)(__ffs(wide) - 1);
            wide &= wide - 1;
            const uint64_t b0 = conv_b(P, t), b1 = conv_b(P, t + 1);
            bool dead;
            const uint32_t nin = t == 0 ? 1u : W.ends[t - 1].n;
            const uint32_t q = t == 0 ? start_state(P, &dead) : W.ends[t - 1].s[lane < nin ? lane : 0];
            uint32_t e = q * T.ES, h = 0;
            bool badseen = false;
            for (uint64_t pos = b0; pos < b1; pos += 32) {
                const uint32_t cnt = (uint32_t)min((uint64_t)32, b1 - pos);
                const uint32_t mine = lane < cnt ? (uint32_t)__ldg(in + pos + lane) : 0u;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, lane < cnt && mine >= d.A);
                if (bal && !badseen) {
                    badseen = true;
                    if (lane == 0) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)(pos + __ffs(bal) - 1));
                }
                for (uint32_t k = 0; k < cnt; ++k) {
                    e = T.next(e, T.col(__shfl_sync(0xFFFFFFFFu, mine, k)));
                    h += T.hit(e);
                }
            }
            // distinct ends of the valid lanes -> this chunk's end set (lane order); every
            // lane takes part in every collective
            const uint32_t e0 = __shfl_sync(0xFFFFFFFFu, e, 0);
            const uint32_t z = lane < nin ? T.state(e) : T.state(e0);
            const uint32_t valid = nin >= 32 ? 0xFFFFFFFFu : ((1u << nin) - 1u);
            const uint32_t m = __match_any_sync(0xFFFFFFFFu, z) & valid;
            const uint32_t first = m ? (uint32_t)(__ffs(m) - 1) : 0u;   // leader of my class
            const uint32_t leaders = __ballot_sync(0xFFFFFFFFu, lane < nin && first == lane);
            const uint32_t idx = __popc(leaders & ((1u << first) - 1u));
            if ((leaders >> lane) & 1u) {
                W.ends[t].s[idx] = z;
                W.surv[t].z[idx] = z;
                W.surv[t].end[idx] = z;
                W.surv[t].tail[idx] = 0;
                W.surv[t].eidx[idx] = (uint8_t)idx;
            }
            if (lane < nin) {
                W.maps[t].idx[lane] = (uint8_t)idx;
                W.maps[t].hits[lane] = h;
            }
            if (lane == 0) {
                W.ends[t].n = __popc(leaders);
                W.surv[t].n = __popc(leaders);
                uint64_t rc = 1;
                if (t > 0) {
                    const uint32_t cl = in[b0 - 1];
                    const uint32_t li = (P.cand == PAREM_CANDIDATES_ENUM || cl >= d.A) ? d.A : cl;
                    rc = route_count(P, cl, in[b0], __ldg(d.Lcnt + li));
                }
                routes += rc;
                steps += rc * (b1 - b0);
            }
            __syncwarp();
        }
    }
    if (lane == 0 && routes) {
        atomicAdd(&P.hdr->routes, routes);
        atomicAdd(&P.hdr->steps, steps);
    }
}

// E2a: chunks entered from ONE possible state (chunk 0, or the previous chunk's routes all
// merged) -- thread per chunk: head walk, survivor pick, validation, stats.
template <bool W32>
__global__ void __launch_bounds__(kFollowThreads) conv_map1_kernel(const MatchParams P) {
    __shared__ unsigned long long acc[3];
    const DevDfa& d = P.d;
    if (threadIdx.x < 3) acc[threadIdx.x] = 0;
    __syncthreads();
    const ConvWs W = conv_ws(P);
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t A = d.A;
    unsigned long long rc = 0, steps = 0, lkm = 0;
    if (t < P.p && W.info[t].D != kWide && (t == 0 || W.ends[t - 1].n == 1)) {
        const uint64_t b0 = conv_b(P, t), b1 = conv_b(P, t + 1);
        const ConvChunk& c = W.info[t];
        const SurvRec& s = W.surv[t];
        bool dead;
        const uint32_t q = t == 0 ? start_state(P, &dead) : W.ends[t - 1].s[0];
        uint32_t hh = 0;
        const uint32_t z = walk1<W32>(d, P.in, b0, b0 + c.m, q, &hh);
        uint32_t k = 0;
        while (k < s.n && s.z[k] != z) ++k;
        if (k == s.n) {
            atomicOr(&P.hdr->err, kErrUnsound);   // speculation unsound: cannot happen
            k = 0;
        }
        W.maps[t].idx[0] = s.eidx[k];
        W.maps[t].hits[0] = hh + s.tail[k];
        const uint64_t off = first_bad(P.in, b0, b0 + c.m, A);   // open chunks: m = whole chunk
        if (off < b0 + c.m) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)off);
        rc = 1;   // stats: |R_t| (R_0 = {q0}) and |R_t| * len_t
        if (t > 0) {
            const uint32_t cl = P.in[b0 - 1];
            const uint32_t li = (P.cand == PAREM_CANDIDATES_ENUM || cl >= A) ? A : cl;
            rc = route_count(P, cl, P.in[b0], __ldg(d.Lcnt + li));
        }
        steps = rc * (b1 - b0);
        lkm = c.m;
    }
    rc = warp_sum(rc);
    steps = warp_sum(steps);
    lkm = warp_sum(lkm);
    if ((threadIdx.x & 31u) == 0 && rc) {
        atomicAdd(acc + 0, rc);
        atomicAdd(acc + 1, steps);
        atomicAdd(acc + 2, lkm);
    }
    __syncthreads();
    if (threadIdx.x == 0 && acc[0]) {
        atomicAdd(&P.hdr->routes, acc[0]);
        atomicAdd(&P.hdr->steps, acc[1]);
        atomicAdd(&P.hdr->lookups, acc[2]);
    }
}

// E2b: chunks entered from SEVERAL possible states (the previous chunk's survivors did not
// merge) -- warp per chunk, lane j walks the head from end-set state j over the same bytes.
template <bool SMEM, bool W32>
__global__ void __launch_bounds__(kSetWarps * 32) conv_map_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ unsigned long long acc[3];
    const DevDfa& d = P.d;
    Tab<SMEM, W32> T;
    T.init(d, stage_table<SMEM, W32>(d, sm));
    if (threadIdx.x < 3) acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const ConvWs W = conv_ws(P);
    const uint8_t* in = P.in;
    const uint32_t A = d.A;
    unsigned long long routes = 0, steps = 0, lkw = 0;
    for (uint64_t t = (uint64_t)blockIdx.x * kSetWarps + warp; t < P.p; t += (uint64_t)gridDim.x * kSetWarps) {
        if (t == 0 || W.info[t].D == kWide) continue;   // wide: conv_wide_kernel's
        const uint32_t nin = W.ends[t - 1].n;
        if (nin <= 1) continue;   // conv_map1_kernel's
        const uint64_t b0 = conv_b(P, t), b1 = conv_b(P, t + 1);
        const ConvChunk& c = W.info[t];
        const SurvRec& s = W.surv[t];
        const uint64_t hb = b0 + c.m;
        const uint32_t q = W.ends[t - 1].s[lane < nin ? lane : 0];
        uint32_t e = q * T.ES, h = 0;
        bool badseen = false;
        for (uint64_t pos = b0; pos < hb; pos += 32) {
            const uint32_t cnt = (uint32_t)min((uint64_t)32, hb - pos);
            const uint32_t mine = lane < cnt ? (uint32_t)__ldg(in + pos + lane) : 0u;
            if (!badseen) {
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, lane < cnt && mine >= A);
                if (bal) {
                    badseen = true;
                    if (lane == 0) atomicMax(&P.hdr->bad_inv, ~(unsigned long long)(pos + __ffs(bal) - 1));
                }
            }
            for (uint32_t k = 0; k < cnt; ++k) {
                e = T.next(e, T.col(__shfl_sync(0xFFFFFFFFu, mine, k)));
                h += T.hit(e);
            }
        }
        if (lane < nin) {
            const uint32_t z = T.state(e);
            uint32_t k = 0;
            while (k < s.n && s.z[k] != z) ++k;
            if (k == s.n) {
                atomicOr(&P.hdr->err, kErrUnsound);   // speculation unsound: cannot happen
                k = 0;
            }
            W.maps[t].idx[lane] = s.eidx[k];
            W.maps[t].hits[lane] = h + s.tail[k];
        }
        if (lane == 0) {   // stats: |R_t| and |R_t| * len_t
            const uint32_t cl = in[b0 - 1];
            const uint32_t li = (P.cand == PAREM_CANDIDATES_ENUM || cl >= A) ? A : cl;
            const uint64_t rc = route_count(P, cl, in[b0], __ldg(d.Lcnt + li));
            routes += rc;
            steps += rc * (b1 - b0);
            lkw += (unsigned long long)nin * c.m;
        }
    }
    if (lane == 0 && routes) {
        atomicAdd(acc + 0, routes);
        atomicAdd(acc + 1, steps);
        atomicAdd(acc + 2, lkw);
    }
    __syncthreads();
    if (threadIdx.x == 0 && acc[0]) {
        atomicAdd(&P.hdr->routes, acc[0]);
        atomicAdd(&P.hdr->steps, acc[1]);
        atomicAdd(&P.hdr->lookups, acc[2]);
    }
}

// E3: compose the maps of each block of kBlk chunks (warp per block, lane = entering index).
__global__ void __launch_bounds__(kFollowThreads) conv_block_kernel(const MatchParams P) {
    const uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nb = (P.p + kBlk - 1) / kBlk;
    if (b >= nb) return;
    const ConvWs W = conv_ws(P);
    const uint64_t c0 = b * kBlk, c1 = min(P.p, c0 + kBlk);
    const uint32_t nin = c0 == 0 ? 1u : W.ends[c0 - 1].n;
    uint32_t idx = lane < nin ? lane : 0;
    for (uint64_t c = c0; c < c1; ++c) idx = W.maps[c].idx[idx];
    W.bmaps[b].idx[lane] = (uint8_t)idx;
}

// E3b: compose the block maps of each super-block of kBlk blocks (warp per super-block).
__global__ void __launch_bounds__(kFollowThreads) conv_super_kernel(const MatchParams P) {
    const uint64_t sb = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nb = (P.p + kBlk - 1) / kBlk, ns = (nb + kBlk - 1) / kBlk;
    if (sb >= ns) return;
    const ConvWs W = conv_ws(P);
    const uint64_t b0 = sb * kBlk, b1 = min(nb, b0 + kBlk);
    const uint64_t c0 = b0 * kBlk;
    const uint32_t nin = c0 == 0 ? 1u : W.ends[c0 - 1].n;
    uint32_t idx = lane < nin ? lane : 0;
    for (uint64_t b = b0; b < b1; ++b) idx = W.bmaps[b].idx[idx];
    W.smaps[sb].idx[lane] = (uint8_t)idx;
}

// E4: one warp walks the super-block maps along q0's path (32 loaded at a time), then
// E4b resolves the entering index of every block (thread per super-block).
__global__ void conv_path_kernel(const MatchParams P) {
    const uint32_t lane = threadIdx.x & 31u;
    if (threadIdx.x >= 32) return;
    const ConvWs W = conv_ws(P);
    const uint64_t nb = (P.p + kBlk - 1) / kBlk, ns = (nb + kBlk - 1) / kBlk;
    uint32_t e = 0;
    for (uint64_t s0 = 0; s0 < ns; s0 += 32) {
        uint32_t v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = s0 + j < ns ? W.smaps[s0 + j].idx[lane] : 0u;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (s0 + j < ns) {
                if (lane == 0) W.sin[s0 + j] = e;
                e = __shfl_sync(0xFFFFFFFFu, v[j], e);
            }
    }
    if (lane == 0) P.hdr->final_q = W.ends[P.p - 1].s[e];
}

__global__ void __launch_bounds__(kFollowThreads) conv_blockin_kernel(const MatchParams P) {
    const uint64_t sb = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nb = (P.p + kBlk - 1) / kBlk, ns = (nb + kBlk - 1) / kBlk;
    if (sb >= ns) return;
    const ConvWs W = conv_ws(P);
    uint32_t e = W.sin[sb];
    const uint64_t b0 = sb * kBlk, b1 = min(nb, b0 + kBlk);
    for (uint64_t b = b0; b < b1; ++b) {
        W.bin[b] = e;
        e = W.bmaps[b].idx[e];
    }
}


// E5: every chunk's entering state and hits (thread per block walking its kBlk maps), the
// total, and the result (last CTA).
__global__ void __launch_bounds__(kFollowThreads) conv_resolve_kernel(const MatchParams P) {
    __shared__ unsigned long long acc;
    __shared__ uint32_t flag;
    if (threadIdx.x == 0) acc = 0;
    __syncthreads();
    const ConvWs W = conv_ws(P);
    const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nb = (P.p + kBlk - 1) / kBlk;
    unsigned long long hits = 0;
    if (b < nb) {
        bool dead;
        const uint32_t q0 = start_state(P, &dead);
        uint32_t e = W.bin[b];
        const uint64_t c0 = b * kBlk, c1 = min(P.p, c0 + kBlk);
        for (uint64_t c = c0; c < c1; ++c) {
            const uint32_t h = W.maps[c].hits[e];
            if (P.fchunk_q) {
                P.fchunk_q[c] = c == 0 ? q0 : W.ends[c - 1].s[e];
                P.fchunk_h[c] = h;
            }
            hits += h;
            e = W.maps[c].idx[e];
        }
    }
    hits = warp_sum(hits);
    if ((threadIdx.x & 31u) == 0 && hits) atomicAdd(&acc, hits);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (acc) atomicAdd(&P.hdr->hits, acc);
        __threadfence();
        flag = atomicAdd(&P.hdr->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!flag || threadIdx.x != 0) return;
    __threadfence();
    const volatile WsHeader* h = P.hdr;
    // internal invariant violated: report instead of a wrong answer -- unless a byte was
    // outside the alphabet (ESYMBOL wins; such a boundary gets a placeholder candidate)
    if ((h->err & kErrUnsound) && h->bad_inv == 0ull) {
        parem_result r;
        memset(&r, 0, sizeof(r));
        r.final_state = PAREM_DEAD;
        r.status = PAREM_EINTERNAL;
        *P.result = r;
        reset_header(P);
        return;
    }
    bool dead;
    start_state(P, &dead);
    write_result(P, h->final_q, h->hits, dead);
}

template <class TT, int CPT>
cudaError_t launch_follow(const Plan& plan, const MatchParams& P, size_t smem, cudaStream_t s) {
    const void* fn = reinterpret_cast<const void*>(&conv_follow_kernel<TT, CPT>);
    cudaError_t e = smem_optin(fn, smem);
    if (e != cudaSuccess) return e;
    if (!TT::kSmem) {
        // global (L2-resident) tables: give the unified L1/shared array to L1 (set once)
        static std::once_flag once;
        std::call_once(once, [fn]() { cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 0); });
    }
    const uint64_t per = (uint64_t)plan.conv_fthreads * CPT;
    const unsigned g = (unsigned)((P.p + per - 1) / per);
    conv_follow_kernel<TT, CPT><<<g, plan.conv_fthreads, smem, s>>>(P);
    return cudaGetLastError();
}

// TMA-staged follow when the input is 16-byte aligned and rows are whole boxes; false =
// not applicable (the caller uses the thread-stream follow)
template <class TT>
bool launch_follow_tma(const MatchParams& P, size_t tb, cudaStream_t s, cudaError_t* err, bool coop = false) {
    if ((((uintptr_t)P.in) & 15u) || P.L % kFBox || P.L < kFBox || P.p < 2) return false;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    if (!coop && !encode_rows_map(&map, P.in, P.L, P.p - 1, kFBox, 32)) return false;
    const void* fn = coop ? reinterpret_cast<const void*>(&conv_follow_tma_kernel<TT, true>)
                          : reinterpret_cast<const void*>(&conv_follow_tma_kernel<TT, false>);
    cudaError_t e = smem_optin(fn, follow_tma_smem(tb));   // tb = the table type's footprint
    if (e == cudaSuccess) {
        void* args[] = {const_cast<MatchParams*>(&P), &map};
        const unsigned g = (unsigned)((P.p + kFThreads - 1) / kFThreads);
        e = cudaLaunchKernel(fn, dim3(g), dim3(kFThreads), args, follow_tma_smem(tb), s);
    }
    *err = e;
    return true;
}

template <class TT>
cudaError_t launch_follow_cpt(const Plan& plan, const MatchParams& P, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (plan.conv_tma && launch_follow_tma<TT>(P, smem, s, &e, plan.conv_tma == 2)) return e;
    return plan.conv_cpt == 2 ? launch_follow<TT, 2>(plan, P, smem, s) : launch_follow<TT, 1>(plan, P, smem, s);
}

template <bool SMEM, bool W32>
int launch_conv_t(const Plan& plan, const MatchParams& P, cudaStream_t s) {
    const DevDfa& d = P.d;
    const size_t tb = smem_tab_bytes(d, SMEM);
    const uint32_t sw = kSetWarps;
    const size_t s1 = tb + sw * set_warp_bytes(P.slots, d.Qpad);
    const bool own = d.Qpad <= kOwnerMaxQ && P.set_own;
    const void* setfn = own ? reinterpret_cast<const void*>(&conv_set_kernel<SMEM, W32, true>)
                            : reinterpret_cast<const void*>(&conv_set_kernel<SMEM, W32, false>);
    cudaError_t e = smem_optin(setfn, s1);
    if (e == cudaSuccess) e = smem_optin(reinterpret_cast<const void*>(&conv_map_kernel<SMEM, W32>), tb);
    int bps = 0, sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, setfn, sw * 32, s1);
    if (bps < 1) bps = 1;
    uint64_t g1w = (P.p + sw - 1) / sw;
    const unsigned g1 = (unsigned)(g1w < (uint64_t)sms * bps ? g1w : (uint64_t)sms * bps);
    const unsigned g2 = (unsigned)((P.p + kFollowThreads - 1) / kFollowThreads);
    {
        void* args[] = {const_cast<MatchParams*>(&P)};
        e = cudaLaunchKernel(setfn, dim3(g1), dim3(sw * 32), args, s1, s);
    }
    prof_after("conv_set", s);
    if constexpr (SMEM) {
        // staged follow (TMA or cooperative cp.async) when the input allows it, else the
        // thread-stream follow -- with the byte-entry table where it applies (the
        // bank-confined u16 copies starve the thread streams' L1)
        const bool coop = plan.conv_tma == 2;
        bool done = false;
        if (plan.conv_tma) {
            if (plan.conv_rep == 8) done = launch_follow_tma<TabR<8>>(P, rep_smem_bytes(d, 8), s, &e, coop);
            else if (plan.conv_rep == 16) done = launch_follow_tma<TabR<16>>(P, rep_smem_bytes(d, 16), s, &e, coop);
            else if (plan.conv_rep == 116 && TabB::applies(d)) done = launch_follow_tma<TabB>(P, TabB::bytes(d), s, &e, coop);
            else done = launch_follow_tma<Tab<SMEM, W32>>(P, tb, s, &e, coop);
        }
        if (!done) {
            const bool byte_tab = TabB::applies(d) && (plan.conv_rep == 116 || (plan.conv_tma && plan.conv_rep != 0));
            if (byte_tab) e = launch_follow<TabB, 1>(plan, P, TabB::bytes(d), s);
            else if (plan.conv_rep == 8 && !plan.conv_tma) e = launch_follow<TabR<8>, 1>(plan, P, rep_smem_bytes(d, 8), s);
            else if (plan.conv_rep == 16 && !plan.conv_tma) e = launch_follow<TabR<16>, 1>(plan, P, rep_smem_bytes(d, 16), s);
            else e = plan.conv_cpt == 2 ? launch_follow<Tab<SMEM, W32>, 2>(plan, P, tb, s)
                                        : launch_follow<Tab<SMEM, W32>, 1>(plan, P, tb, s);
        }
    } else {
        if (plan.conv_hyb && !W32 && TabH::applies(d))
            e = plan.conv_cpt == 2 ? launch_follow<TabH, 2>(plan, P, TabH::bytes(d), s)
                                   : launch_follow<TabH, 1>(plan, P, TabH::bytes(d), s);
        else e = launch_follow_cpt<Tab<SMEM, W32>>(plan, P, tb, s);
    }
    prof_after("conv_follow", s);
    if (e != cudaSuccess) {
        set_error("conv_follow: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    conv_ends_kernel<<<g2, kFollowThreads, 0, s>>>(P);
    prof_after("conv_ends", s);
    conv_wide_kernel<W32><<<1, 32, 0, s>>>(P);
    prof_after("conv_wide", s);

    int bpm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpm, conv_map_kernel<SMEM, W32>, kSetWarps * 32, tb);
    if (bpm < 1) bpm = 1;
    const uint64_t gmw = (P.p + kSetWarps - 1) / kSetWarps;
    const unsigned gm = (unsigned)(gmw < (uint64_t)sms * bpm ? gmw : (uint64_t)sms * bpm);
    conv_map1_kernel<W32><<<g2, kFollowThreads, 0, s>>>(P);
    prof_after("conv_map1", s);
    conv_map_kernel<SMEM, W32><<<gm, kSetWarps * 32, tb, s>>>(P);
    prof_after("conv_map", s);

    const uint64_t nb = (P.p + kBlk - 1) / kBlk;
    conv_block_kernel<<<(unsigned)((nb * 32 + kFollowThreads - 1) / kFollowThreads), kFollowThreads, 0, s>>>(P);
    prof_after("conv_block", s);
    const uint64_t nsb = (nb + kBlk - 1) / kBlk;
    conv_super_kernel<<<(unsigned)((nsb * 32 + kFollowThreads - 1) / kFollowThreads), kFollowThreads, 0, s>>>(P);
    prof_after("conv_super", s);
    conv_path_kernel<<<1, 32, 0, s>>>(P);
    prof_after("conv_path", s);
    conv_blockin_kernel<<<(unsigned)((nsb + kFollowThreads - 1) / kFollowThreads), kFollowThreads, 0, s>>>(P);
    prof_after("conv_blockin", s);
    conv_resolve_kernel<<<(unsigned)((nb + kFollowThreads - 1) / kFollowThreads), kFollowThreads, 0, s>>>(P);
    prof_after("conv_resolve", s);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("conv kernels: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    return PAREM_OK;
}

}  // namespace

size_t conv_ws_total(uint64_t p) { return conv_ws_bytes(p); }

size_t conv_rep_smem(const DevDfa& d, uint32_t R) { return rep_smem_bytes(d, R); }
bool conv_hybrid_applies(const DevDfa& d) { return TabH::applies(d); }
bool conv_byte_table_applies(const DevDfa& d) { return TabB::applies(d); }
size_t conv_follow_tma_smem(size_t table_bytes) { return follow_tma_smem(table_bytes); }

size_t conv_set_smem_bytes(const DevDfa& d, bool smem_tab, uint32_t cap, uint32_t warps) {
    return smem_tab_bytes(d, smem_tab) + warps * set_warp_bytes(cap, d.Qpad);
}

int launch_conv(const Plan& plan, const MatchParams& P, cudaStream_t s) {
    const bool sm = plan.smem_tab != 0, w = P.d.lanes_u32 != 0;
    if (sm && w) return launch_conv_t<true, true>(plan, P, s);
    if (sm && !w) return launch_conv_t<true, false>(plan, P, s);
    if (!sm && w) return launch_conv_t<false, true>(plan, P, s);
    return launch_conv_t<false, false>(plan, P, s);
}

}  // namespace parem
