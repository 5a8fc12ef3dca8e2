// internal.h -- internal types of the PaREM B200 library (not part of the ABI).
//
// Data layout in HBM / shared memory:
//   * the caller's table is turned into a COMPLETE internal table over Qp = Q (+1 sink if
//     any entry is DEAD): DEAD -> sink, sink -> sink, sink not accepting (reading C9);
//   * L(c) lists (sorted, over the original Q, DEAD excluded: P:67) for every
//     symbol, plus list A = all of Q (Enum candidates);
//   * tiny class (Qp <= 32): tab1[s][c] = dest | acc(dest) << 15 (u16) and, for A <= 4,
//     the 4-bit-group stride table stride[s][g] = dest << 11 | hits << 28 (g packs
//     4/B symbols of B bits, earliest symbol in the low bits);
//   * lanes class (Qp > 32): symbol-major tabL[c][s] over Apad x Qpad (powers of two),
//     entry = dest * ES | acc(dest) << (8*ES - 1) with ES = 2 (u16) or 4 (u32) bytes, so
//     the next byte offset is (entry & SMASK) | (c << SHC) -- one LOP3 per lookup.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <vector>

#include "parem.h"

namespace parem {

constexpr uint32_t kTinyMaxStates = 32;   // dense per-chunk maps live in one warp
constexpr uint32_t kTinyThreads = 512;    // threads per CTA, tiny kernel
constexpr uint32_t kTinyRowsPerThread = 2;  // chunks per thread, tiny kernel
constexpr uint32_t kTinyMaxA = 256;
constexpr uint32_t kKernelTrivial = 0, kKernelTiny = 1, kKernelLanes = 2, kKernelConv = 3;

struct DevDfa {                // POD, passed by value to every kernel
    uint32_t Q, Qp, Qpad, A;
    uint32_t Apad, sink, start, has_sink;
    uint32_t log2Qpad, Lmin, Lmax, sym_bits;   // sym_bits: 0 (no stride table), 1, 2
    uint32_t lanes_u32, Lsum_all, pad0, pad1;  // Lsum_all = total list entries incl. list A
    const uint8_t* acc;        // [Qp] accept flag per internal state
    const uint32_t* Loff;      // [A+1]
    const uint32_t* Lcnt;      // [A+1]
    const uint32_t* Llist;     // concatenated lists
    const uint32_t* Rcnt;      // [A*A] |L(a) n S(b)| (partial tables only), else nullptr
    const uint16_t* tab1;      // tiny: [Qp][A]
    const uint32_t* stride;    // tiny: [Qp][16]
    const void* lanes_tab;     // lanes: [Apad][Qpad]
};

struct WsHeader {              // first 64 bytes of every workspace (memset to 0 per call)
    unsigned int done;         // CTAs finished (last-CTA detection)
    unsigned int err;          // conv path: internal invariant violated
    unsigned long long bad_inv;  // ~(smallest bad local offset); 0 = none
    unsigned long long routes;   // sum |R_i|
    unsigned long long steps;    // sum |R_i| * len_i
    unsigned long long hits;     // conv path: total hits along the true path
    unsigned int final_q;        // conv path: state after the last chunk
    unsigned int pad;
    unsigned long long lookups;  // conv path: table lookups issued at distinct states (set walk:
                                 // the deduplicated set per step; follow / head walks: live routes)
    unsigned long long pad2;
};
static_assert(sizeof(WsHeader) == 64, "header");

struct MatchParams {
    DevDfa d;
    const uint8_t* in;
    uint64_t n;
    uint64_t L;                // nominal chunk length
    uint64_t p;                // number of chunks
    uint32_t policy, cand, win, slots;
    uint32_t tg;               // lanes: threads per chunk group
    uint32_t stages;           // tiny: TMA stages per warp (0 = no TMA)
    uint32_t dmax;             // conv: survivors handed from the set walk to the follow walk
    uint32_t lookback;         // tiny: k of the look-back candidate rule
    uint32_t conv_cpt;         // conv: chunks per follow thread
    uint32_t set_own;          // conv: phase-A dedup by owner tags (else image bitmap + atomics)
    // parem_match_batch_async (tiny kernel): `batch` independent inputs of n_one bytes laid
    // out back to back; chunk t belongs to input t / cpi (cpi = a multiple of the CTA tile)
    uint64_t cpi;              // chunks per input (0 = not a batch)
    uint64_t n_one;            // bytes per input
    parem_result* results;     // [batch] per-input results
    unsigned long long* bstats;  // [batch][4]: ~bad offset (local), routes, steps, pad
    uint64_t offset_base;
    const parem_result* carry; // may be null
    parem_result* result;
    WsHeader* hdr;
    void* maps;                // tiny: tile maps [grid][Qpad] u64; lanes: ends [p][Qpad] u32 + hits
    uint32_t* map_hits;        // lanes only
    // parem_find_async (NEXT-4; kernels_find.cu): null for a plain match
    uint32_t* tout;            // parem_trace_async: visited states of the window [tlo, thi)
    uint64_t tlo, thi;
    uint64_t* fout;            // match end offsets
    uint64_t fmax;             // capacity of fout
    uint32_t* fchunk_q;        // [p] entering state of chunk i
    uint32_t* fchunk_h;        // [p] hits of chunk i from that state
    unsigned long long* fchunk_base;   // [p] exclusive prefix of fchunk_h
    unsigned long long* fblock;        // scan block sums
    uint32_t* fgq;             // tiny: entering state per group of 32 chunks
    uint8_t* fmend;            // tiny: per-chunk dense maps (end) [p][Qpad]
    uint32_t* fmhits;          // tiny: per-chunk dense maps (hits) [p][Qpad]
    uint32_t* fgend;           // tiny: per-group maps (end) [groups][Qpad]
    unsigned long long* fghits;        // tiny: per-group maps (hits)
    uint32_t* fsend;           // tiny: per-super-group maps (end) [groups/32][Qpad]
    uint32_t* fsq;             // tiny: entering state per super-group
};

struct Plan {
    uint32_t kernel;
    uint32_t threads;
    uint64_t grid;
    uint64_t p, L;
    uint32_t policy, cand, slots, U;
    uint32_t tg;             // lanes: threads per chunk group (blockDim = G * tg)
    uint32_t sym_per_lookup;
    uint32_t win;
    uint32_t smem_tab;       // lanes: table staged in shared memory
    uint32_t tma;            // tiny: TMA stages per warp (0 = rows read with 16-B loads)
    uint32_t dmax;           // conv: set-walk hand-over threshold (1, 2 or 4 survivors)
    uint32_t conv_tma;       // conv: TMA-staged follow walk (rows of L bytes)
    uint32_t conv_rep;       // conv: follow table replicated in R = 8 / 16 copies (0: plain)
    uint32_t conv_hyb;       // conv: hybrid follow table (packed columns in shared memory + L2)
    uint32_t set_own;        // conv: phase-A dedup by owner tags (Qpad <= 1024)
    uint32_t conv_cpt;       // conv: chunks per follow thread (1 or 2)
    uint32_t conv_fthreads;  // conv: follow block size
    uint32_t conv_swarps;    // conv: set-walk warps per CTA
    size_t smem;
    size_t ws;
    size_t off_maps, off_hits;
};

}  // namespace parem

struct parem_dfa {
    parem::DevDfa dev;
    uint32_t Q, A, start, eb;
    uint32_t Lmin, Lmax;
    uint64_t Lsum;
    uint32_t table_class;
    int device;
    void* dev_block;
    size_t dev_bytes;
    int num_sms;
    // create-time convergence probe (set walk from all of Q under seeded uniform symbols):
    // steps until <= 4 / exactly 1 distinct states remain (0 = not within the probe)
    uint32_t conv_t4, conv_t1;
    uint64_t conv_work4;
};

namespace parem {
// host side (dfa.cpp / planner.cpp / abi.cu)
void set_error(const char* fmt, ...);
// per-kernel timing (parem_profile): call after each kernel launch of a match
void prof_after(const char* name, cudaStream_t s);
// Raise a kernel's dynamic shared memory limit to at least `bytes`, under a mutex, never
// lowering it: the attribute is process-wide, so a concurrent match on another host thread
// can never see it drop below what its own launch needs.  Keeping it at the
// largest size actually launched (rather than the opt-in maximum) leaves the driver's
// shared/L1 carveout choice to the real footprint.
cudaError_t smem_optin(const void* fn, size_t bytes);
int make_plan(const parem_dfa* dfa, uint64_t n, const parem_options* opts, Plan* plan);
// device side (kernels_*.cu)
int launch_tiny(const Plan& plan, const MatchParams& P, cudaStream_t s);
int launch_lanes(const Plan& plan, const MatchParams& P, cudaStream_t s);
int launch_conv(const Plan& plan, const MatchParams& P, cudaStream_t s);
int launch_find(const Plan& plan, const MatchParams& P, cudaStream_t s);
size_t find_extra_bytes(const Plan& plan, const DevDfa& d);
void find_bind(const Plan& plan, MatchParams& P, unsigned char* extra);
size_t conv_ws_total(uint64_t p);
size_t conv_rep_smem(const DevDfa& d, uint32_t R);        // 0 if the layout does not apply
bool conv_hybrid_applies(const DevDfa& d);
bool conv_byte_table_applies(const DevDfa& d);
size_t conv_follow_tma_smem(size_t table_bytes);
size_t conv_set_smem_bytes(const DevDfa& d, bool smem_tab, uint32_t cap, uint32_t warps);
int launch_trivial(const MatchParams& P, cudaStream_t s);
int launch_segment_head(const DevDfa& d, const uint8_t* in, uint64_t X, const uint32_t* cand, uint32_t ncand,
                        uint32_t* st_out, unsigned long long* hits_out, unsigned long long* bad_inv, cudaStream_t s);
bool encode_rows_map(CUtensorMap* map, const uint8_t* base, uint64_t row_len, uint64_t rows, uint32_t box_w,
                     uint32_t box_rows);
int tiny_blocks_per_sm(uint32_t K, uint32_t B, bool tma, size_t smem);
size_t tiny_smem_bytes(const DevDfa& d, uint32_t B, uint32_t stages);
uint32_t tiny_pick_stages(const DevDfa& d, uint32_t B);
size_t lanes_smem_bytes(const DevDfa& d, bool smem_tab);
int lanes_blocks_per_sm(uint32_t U, bool smem_tab, bool u32, uint32_t threads, size_t smem);
uint32_t tiny_round_slots(uint32_t k, uint32_t B);
uint32_t lanes_max_groups();
}  // namespace parem
