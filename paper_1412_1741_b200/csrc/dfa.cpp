// dfa.cpp -- DFA ingest: validation, the complete internal table
// with a DEAD sink, the per-symbol L(c) lists and S-intersection counts, the tiny/lanes
// device tables, and the single device upload.  Host code only.
//
// Paper: DFA quintuple; transition table Tt as an adjacency matrix;
// S(c) / L(c) (Alg. 1 lines 5-14; reading C1: L on the previous chunk's last
// symbol); the paper recomputes S and L per chunk in O(|Q|) -- precomputing them per
// symbol once is equivalent (they depend only on the symbol).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "internal.h"

namespace parem {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static uint32_t pow2_at_least(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

static uint32_t log2u(uint32_t p) {
    uint32_t l = 0;
    while ((1u << l) < p) ++l;
    return l;
}

}  // namespace parem

using namespace parem;

extern "C" const char* parem_last_error(void) { return g_err; }
extern "C" const char* parem_version(void) { return "parem-b200 0.1 (sm_100a)"; }

extern "C" int parem_dfa_create(uint32_t Q, uint32_t A, const void* table, uint32_t eb, uint32_t start,
                                const uint8_t* accept_bitmap, parem_dfa** out) {
    set_error("");
    if (!out || !table || !accept_bitmap) { set_error("null argument"); return PAREM_EINVAL; }
    if (Q == 0) { set_error("num_states must be >= 1"); return PAREM_EINVAL; }
    if (A == 0 || A > 256) { set_error("alphabet_size must be in [1, 256]"); return PAREM_EINVAL; }
    if (eb != 2 && eb != 4) { set_error("elem_bytes must be 2 or 4"); return PAREM_EINVAL; }
    if (eb == 2 && Q > 65535) { set_error("uint16 tables need num_states <= 65535"); return PAREM_EINVAL; }
    // device table offsets are u32 (symbol-major lanes table: Apad * Qpad * 4 bytes < 2^32)
    // and the accept bit sits above dest * 4 in a u32 entry: Q <= 2^22 keeps both exact
    if (Q > (1u << 22)) { set_error("num_states %u > 4194304 is not supported", Q); return PAREM_EINVAL; }
    if (start >= Q) { set_error("start_state %u >= num_states %u", start, Q); return PAREM_EINVAL; }
    const uint32_t dead_in = eb == 2 ? 0xFFFFu : 0xFFFFFFFFu;

    // ---- validation + complete internal table (row-major [Qp][A], u32) ----
    bool has_sink = false;
    const uint64_t QA = (uint64_t)Q * A;
    for (uint64_t i = 0; i < QA; ++i) {
        uint32_t v = eb == 2 ? ((const uint16_t*)table)[i] : ((const uint32_t*)table)[i];
        if (v == dead_in) { has_sink = true; continue; }
        if (v >= Q) {
            set_error("table[%llu] = %u is neither < num_states nor DEAD", (unsigned long long)i, v);
            return PAREM_EINVAL;
        }
    }
    const uint32_t Qp = Q + (has_sink ? 1 : 0);
    const uint32_t sink = has_sink ? Q : 0xFFFFFFFFu;
    std::vector<uint32_t> tab((size_t)Qp * A);
    for (uint64_t i = 0; i < QA; ++i) {
        uint32_t v = eb == 2 ? ((const uint16_t*)table)[i] : ((const uint32_t*)table)[i];
        tab[i] = v == dead_in ? sink : v;
    }
    if (has_sink)
        for (uint32_t c = 0; c < A; ++c) tab[(size_t)sink * A + c] = sink;
    std::vector<uint8_t> acc(Qp, 0);
    for (uint32_t s = 0; s < Q; ++s) acc[s] = (accept_bitmap[s >> 3] >> (s & 7)) & 1;

    // ---- L(c) lists: sorted unique destinations over original Q, DEAD excluded ----
    std::vector<uint32_t> Loff(A + 1), Lcnt(A + 1), Llist;
    std::vector<uint8_t> mark(Qp);
    uint32_t Lmin = 0xFFFFFFFFu, Lmax = 0;
    uint64_t Lsum = 0;
    for (uint32_t c = 0; c < A; ++c) {
        std::fill(mark.begin(), mark.end(), 0);
        for (uint32_t q = 0; q < Q; ++q) {
            uint32_t d = tab[(size_t)q * A + c];
            if (d != sink) mark[d] = 1;
        }
        Loff[c] = (uint32_t)Llist.size();
        for (uint32_t q = 0; q < Q; ++q)
            if (mark[q]) Llist.push_back(q);
        Lcnt[c] = (uint32_t)Llist.size() - Loff[c];
        Lmin = std::min(Lmin, Lcnt[c]);
        Lmax = std::max(Lmax, Lcnt[c]);
        Lsum += Lcnt[c];
    }
    Loff[A] = (uint32_t)Llist.size();     // list A: all of Q (Enum)
    for (uint32_t q = 0; q < Q; ++q) Llist.push_back(q);
    Lcnt[A] = Q;

    // ---- Rcnt[a][b] = |L(a) n S(b)| for partial tables (stats only) ----
    std::vector<uint32_t> Rcnt;
    if (has_sink) {
        Rcnt.assign((size_t)A * A, 0);
        const uint32_t words = (Q + 63) / 64;
        std::vector<uint64_t> Sbits((size_t)A * words, 0), Lbits((size_t)A * words, 0);
        for (uint32_t q = 0; q < Q; ++q)
            for (uint32_t c = 0; c < A; ++c) {
                uint32_t d = tab[(size_t)q * A + c];
                if (d != sink) {
                    Sbits[(size_t)c * words + q / 64] |= 1ull << (q % 64);
                    Lbits[(size_t)c * words + d / 64] |= 1ull << (d % 64);
                }
            }
        for (uint32_t a = 0; a < A; ++a)
            for (uint32_t b = 0; b < A; ++b) {
                uint32_t cnt = 0;
                for (uint32_t w = 0; w < words; ++w)
                    cnt += (uint32_t)__builtin_popcountll(Lbits[(size_t)a * words + w] & Sbits[(size_t)b * words + w]);
                Rcnt[(size_t)a * A + b] = cnt;
            }
    }

    // ---- class-specific tables ----
    const bool tiny = Qp <= kTinyMaxStates;
    uint32_t sym_bits = 0;
    std::vector<uint16_t> tab1;
    std::vector<uint32_t> stride;
    std::vector<uint8_t> lanes;   // raw bytes
    uint32_t Qpad = pow2_at_least(Qp), Apad = pow2_at_least(A);
    bool lanes_u32 = false;
    if (tiny) {
        tab1.resize((size_t)Qp * A);
        for (uint32_t s = 0; s < Qp; ++s)
            for (uint32_t c = 0; c < A; ++c) {
                uint32_t d = tab[(size_t)s * A + c];
                tab1[(size_t)s * A + c] = (uint16_t)(d | (acc[d] << 15));
            }
        if (A <= 4) {
            sym_bits = A <= 2 ? 1 : 2;
            if (A == 3) sym_bits = 0;   // non-power-of-two: generic path (exact byte checks)
        }
        if (sym_bits) {
            const uint32_t KS = 4 / sym_bits, mask = (1u << sym_bits) - 1;
            stride.resize((size_t)Qp * 16);
            for (uint32_t s = 0; s < Qp; ++s)
                for (uint32_t g = 0; g < 16; ++g) {
                    uint32_t st = s, hits = 0;
                    for (uint32_t j = 0; j < KS; ++j) {
                        uint32_t c = (g >> (sym_bits * j)) & mask;   // earliest symbol lowest
                        if (c >= A) c = 0;  // code only produced by invalid bytes (ESYMBOL)
                        st = tab[(size_t)st * A + c];
                        hits += acc[st];
                    }
                    stride[(size_t)s * 16 + g] = (st << 11) | (hits << 28);
                }
        }
    } else {
        // u32 entries when the table is staged in shared memory (32-bit LDS takes the
        // [reg + uniform base] form) or when dest*2 no longer fits 15 bits
        lanes_u32 = Qpad > 16384 || (size_t)Apad * Qpad * 4 <= (size_t)160 * 1024;
        const uint32_t ES = lanes_u32 ? 4 : 2;
        lanes.assign((size_t)Apad * Qpad * ES, 0);
        for (uint32_t c = 0; c < A; ++c)
            for (uint32_t s = 0; s < Qp; ++s) {
                uint32_t d = tab[(size_t)s * A + c];
                size_t i = (size_t)c * Qpad + s;
                if (lanes_u32) ((uint32_t*)lanes.data())[i] = d * 4u | ((uint32_t)acc[d] << 31);
                else ((uint16_t*)lanes.data())[i] = (uint16_t)(d * 2u | ((uint32_t)acc[d] << 15));
            }
    }

    // ---- one device allocation for everything ----
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t o_acc = 0, o_loff = al(o_acc + Qp), o_lcnt = al(o_loff + 4 * (A + 1)),
           o_llist = al(o_lcnt + 4 * (A + 1)), o_rcnt = al(o_llist + 4 * Llist.size()),
           o_tab1 = al(o_rcnt + 4 * Rcnt.size()), o_stride = al(o_tab1 + 2 * tab1.size()),
           o_lanes = al(o_stride + 4 * stride.size()), total = al(o_lanes + lanes.size());
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { set_error("no CUDA device"); return PAREM_ECUDA; }
    void* blk = nullptr;
    cudaError_t e = cudaMalloc(&blk, total);
    if (e != cudaSuccess) { set_error("cudaMalloc(%zu): %s", total, cudaGetErrorString(e)); return PAREM_ENOMEM; }
    std::vector<uint8_t> host(total, 0);
    memcpy(&host[o_acc], acc.data(), Qp);
    memcpy(&host[o_loff], Loff.data(), 4 * (A + 1));
    memcpy(&host[o_lcnt], Lcnt.data(), 4 * (A + 1));
    memcpy(&host[o_llist], Llist.data(), 4 * Llist.size());
    if (!Rcnt.empty()) memcpy(&host[o_rcnt], Rcnt.data(), 4 * Rcnt.size());
    if (!tab1.empty()) memcpy(&host[o_tab1], tab1.data(), 2 * tab1.size());
    if (!stride.empty()) memcpy(&host[o_stride], stride.data(), 4 * stride.size());
    if (!lanes.empty()) memcpy(&host[o_lanes], lanes.data(), lanes.size());
    e = cudaMemcpy(blk, host.data(), total, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(blk);
        set_error("cudaMemcpy: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }

    // ---- convergence probe for the converging path (kernels_conv.cu): the set walk
    // delta*(Q, w) under seeded uniform symbols; how many steps until <= 4 / 1 states ----
    uint32_t conv_t4 = 0, conv_t1 = 0;
    uint64_t conv_work4 = 0;   // sum of set sizes until <= 4 states: the set walk's lookups per chunk
    if (!tiny && !has_sink) {
        std::vector<uint32_t> cur(Qp), nxt;
        std::vector<uint32_t> mark(Qp, 0);
        for (uint32_t s = 0; s < Qp; ++s) cur[s] = s;
        uint64_t x = 0x9E3779B97F4A7C15ull;
        // bounded by total work (<= 2^27 lookups): a DFA whose routes never merge (e.g.
        // permutation columns) ends the probe early and stays off the converging path
        uint64_t work = 0;
        for (uint32_t t = 1; t <= (1u << 16) && cur.size() > 1 && work < (1ull << 27); ++t) {
            work += cur.size();
            x += 0x9E3779B97F4A7C15ull;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            const uint32_t c = (uint32_t)(((unsigned __int128)z * A) >> 64);
            nxt.clear();
            for (uint32_t s : cur) {
                const uint32_t d2 = tab[(size_t)s * A + c];
                if (mark[d2] != t) {
                    mark[d2] = t;
                    nxt.push_back(d2);
                }
            }
            cur.swap(nxt);
            if (!conv_t4 && cur.size() <= 4) {
                conv_t4 = t;
                conv_work4 = work;
            }
            if (cur.size() == 1) conv_t1 = t;
        }
    }

    parem_dfa* h = new parem_dfa();
    DevDfa& d = h->dev;
    memset(&d, 0, sizeof(d));
    char* b = (char*)blk;
    d.Q = Q; d.Qp = Qp; d.Qpad = Qpad; d.A = A; d.Apad = Apad; d.sink = sink; d.start = start;
    d.has_sink = has_sink; d.log2Qpad = log2u(Qpad); d.Lmin = Lmin; d.Lmax = Lmax; d.sym_bits = sym_bits;
    d.lanes_u32 = lanes_u32; d.Lsum_all = (uint32_t)Llist.size();
    d.acc = (const uint8_t*)(b + o_acc);
    d.Loff = (const uint32_t*)(b + o_loff);
    d.Lcnt = (const uint32_t*)(b + o_lcnt);
    d.Llist = (const uint32_t*)(b + o_llist);
    d.Rcnt = Rcnt.empty() ? nullptr : (const uint32_t*)(b + o_rcnt);
    d.tab1 = tab1.empty() ? nullptr : (const uint16_t*)(b + o_tab1);
    d.stride = stride.empty() ? nullptr : (const uint32_t*)(b + o_stride);
    d.lanes_tab = lanes.empty() ? nullptr : (const void*)(b + o_lanes);
    h->Q = Q; h->A = A; h->start = start; h->eb = eb;
    h->Lmin = Lmin; h->Lmax = Lmax; h->Lsum = Lsum;
    h->table_class = tiny ? 1 : (lanes.size() <= (size_t)160 * 1024 ? 2 : 3);
    h->device = dev;
    h->dev_block = blk;
    h->dev_bytes = total;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    h->num_sms = sms;
    h->conv_t4 = conv_t4;
    h->conv_t1 = conv_t1;
    h->conv_work4 = conv_work4;
    *out = h;
    return PAREM_OK;
}

extern "C" int parem_dfa_destroy(parem_dfa* dfa) {
    if (!dfa) return PAREM_OK;
    cudaError_t e = cudaFree(dfa->dev_block);
    delete dfa;
    if (e != cudaSuccess) { set_error("cudaFree: %s", cudaGetErrorString(e)); return PAREM_ECUDA; }
    return PAREM_OK;
}

extern "C" int parem_dfa_get_info(const parem_dfa* dfa, parem_dfa_info* info) {
    if (!dfa || !info) { set_error("null argument"); return PAREM_EINVAL; }
    memset(info, 0, sizeof(*info));
    info->num_states = dfa->Q;
    info->internal_states = dfa->dev.Qp;
    info->alphabet_size = dfa->A;
    info->has_sink = dfa->dev.has_sink;
    info->min_L = dfa->Lmin;
    info->max_L = dfa->Lmax;
    info->sum_L = dfa->Lsum;
    info->start_state = dfa->start;
    info->table_class = dfa->table_class;
    info->device_bytes = dfa->dev_bytes;
    return PAREM_OK;
}
