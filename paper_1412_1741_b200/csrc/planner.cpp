// planner.cpp -- the chunk-size / candidate-set planner (north_star
// subsystem (3)).  It trades redundant work against parallelism:
//   * the paper splits into p = #processing units chunks of T.length/p;
//     on a GPU "processing units" are register slots / lanes, so the default is ONE wave
//     of resident CTAs (every thread/CTA gets exactly one chunk; no tail effect);
//   * redundant work is sum_i (|R_i| - 1) * len_i; the SNAP policy moves each nominal
//     boundary forward (<= win bytes) to a position whose preceding symbol minimises
//     |L(c)|, so the tiny kernel can size its register slots for min_c |L(c)| instead of
//     max_c |L(c)| (W_exec <= W_grid; results are partition-invariant);
//   * slots (registers per thread, or lanes per CTA) are sized for the expected |R_i|;
//     a chunk with more candidates runs extra passes over its bytes.
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <tuple>

#include "internal.h"

namespace parem {

static int cached_bps(int kind, uint32_t a, uint32_t b, uint32_t c, uint32_t threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, uint32_t, uint32_t, uint32_t, uint32_t, size_t, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    auto key = std::make_tuple(kind, a, b, c, threads, smem, dev);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int v = kind == 1 ? tiny_blocks_per_sm(a, b, c != 0, smem) : lanes_blocks_per_sm(a, b != 0, c != 0, threads, smem);
    std::lock_guard<std::mutex> g(mu);
    cache[key] = v;
    return v;
}

static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Tiny kernel: the remainder r = n mod L is walked by the last chunk's thread after its
// row (reading C7), ~0.7x the time per byte of the streamed rows; longer rows cost every
// thread.  Among the row lengths L0, L0 + 64, ... (not multiples of 256 B, see
// profiles/r01_stride_probe.txt) take the one minimising 3 L + 2 r.
static uint64_t pick_row_len(uint64_t n, uint64_t L0) {
    uint64_t best = L0, best_cost = ~0ull;
    for (uint64_t j = 0; j < 64; ++j) {
        const uint64_t L = L0 + 64 * j;
        if (L > n) break;
        if (L % 256 == 0) continue;
        const uint64_t cost = 3 * L + 2 * (n % L);
        if (cost < best_cost) {
            best_cost = cost;
            best = L;
        }
    }
    return best;
}
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

int make_plan(const parem_dfa* dfa, uint64_t n, const parem_options* opts, Plan* plan) {
    memset(plan, 0, sizeof(*plan));
    if (!dfa) { set_error("null dfa"); return PAREM_EINVAL; }
    const DevDfa& d = dfa->dev;
    uint32_t policy = opts ? opts->boundary_policy : PAREM_BOUNDARY_AUTO;
    const uint32_t cand = opts ? opts->candidates : PAREM_CANDIDATES_PAREM;
    const uint32_t kreq = opts ? opts->kernel : 0;
    const uint64_t forced = opts ? opts->chunk_len : 0;
    if (policy > PAREM_BOUNDARY_AUTO) { set_error("bad boundary_policy %u", policy); return PAREM_EINVAL; }
    if (cand > PAREM_CANDIDATES_LOOKBACK) { set_error("bad candidates %u", cand); return PAREM_EINVAL; }
    if (cand == PAREM_CANDIDATES_LOOKBACK && (!opts || opts->lookback == 0)) {
        set_error("look-back candidates need options.lookback >= 1");
        return PAREM_EINVAL;
    }
    if (kreq > kKernelConv) { set_error("bad kernel %u", kreq); return PAREM_EINVAL; }
    plan->cand = cand;
    if (n == 0) {
        plan->policy = policy == PAREM_BOUNDARY_AUTO ? PAREM_BOUNDARY_GRID : policy;
        plan->kernel = kKernelTrivial;
        plan->threads = 32;
        plan->grid = 1;
        plan->ws = 256;
        return PAREM_OK;
    }
    // converging path: complete tables whose routes merge (create-time probe), |Q| small
    // enough for u16 candidate lists and the set walk's per-warp scratch
    const uint32_t conv_cap = cand == PAREM_CANDIDATES_ENUM ? d.Q : d.Lmax;
    const bool conv_smem_tab = d.lanes_tab && (size_t)d.Apad * d.Qpad * (d.lanes_u32 ? 4 : 2) <= (size_t)160 * 1024;
    const uint32_t conv_swarps = 8;   // set-walk warps per CTA
    const bool conv_ok = d.lanes_tab && !d.has_sink && d.Qpad <= 65536 && dfa->conv_t4 > 0 &&
                         conv_set_smem_bytes(d, conv_smem_tab, conv_cap, conv_swarps) <= (size_t)200 * 1024;
    uint32_t kernel = kreq ? kreq
                           : (d.Qp <= kTinyMaxStates ? kKernelTiny : (conv_ok ? kKernelConv : kKernelLanes));
    if (kernel == kKernelConv && !conv_ok) {
        set_error("converging path needs a complete table of <= 65536 states whose routes merge");
        return PAREM_EINVAL;
    }
    if (cand == PAREM_CANDIDATES_LOOKBACK && kernel != kKernelTiny) {
        set_error("look-back candidates are implemented by the tiny kernel (<= %u states)", kTinyMaxStates);
        return PAREM_EINVAL;
    }
    if (kernel == kKernelTiny && d.Qp > kTinyMaxStates) {
        set_error("tiny kernel needs <= %u internal states (have %u)", kTinyMaxStates, d.Qp);
        return PAREM_EINVAL;
    }
    if (kernel == kKernelLanes && !d.lanes_tab) {
        set_error("lanes kernel needs a lanes table (DFA has <= %u states)", kTinyMaxStates);
        return PAREM_EINVAL;
    }
    plan->kernel = kernel;
    // AUTO: the thread-per-chunk kernel merges converged routes, so the paper's own GRID
    // partition costs little extra when every |L(c)| fits the register slots;
    // SNAP (shorter candidate lists, but boundary scans and unaligned heads) otherwise.
    if (policy == PAREM_BOUNDARY_AUTO)
        policy = (kernel == kKernelTiny && d.Lmax <= 8) ? PAREM_BOUNDARY_GRID : PAREM_BOUNDARY_SNAP;
    plan->policy = policy;
    const int sms = dfa->num_sms > 0 ? dfa->num_sms : 148;

    if (kernel == kKernelTiny) {
        const uint32_t B = d.sym_bits;
        // look-back sets are at most |L(c)|; from k >= 4 on usually far smaller (size for the
        // smallest |L(c)|, extra passes cover the rest)
        const bool lb_small = cand == PAREM_CANDIDATES_LOOKBACK && opts->lookback >= 4;
        uint32_t need = cand == PAREM_CANDIDATES_ENUM ? d.Q
                        : (lb_small || policy == PAREM_BOUNDARY_SNAP) ? d.Lmin : d.Lmax;
        if (need < 1) need = 1;
        const uint32_t K = tiny_round_slots(need, B);
        const uint32_t stages = (forced == 0 || forced % 64 == 0) ? tiny_pick_stages(d, B) : 0u;
        const size_t smem = tiny_smem_bytes(d, B, stages);
        int bps = cached_bps(1, K, B, stages, kTinyThreads, smem);
        if (bps <= 0) { set_error("tiny kernel does not fit (smem %zu)", smem); return PAREM_EINVAL; }
        uint64_t L;
        if (forced) L = forced;
        else {
            const uint64_t target = (uint64_t)sms * bps * kTinyThreads * kTinyRowsPerThread;
            L = ceil_div(n, target);
            L = (L + 63) & ~63ull;       // whole TMA boxes per row
            if (L < 64) L = 64;   // one TMA box per row: small inputs still spread over many CTAs
            L = pick_row_len(n, L);
        }
        plan->tma = stages;
        if (L > (1ull << 30)) L = 1ull << 30;
        const uint64_t p = n / L ? n / L : 1;
        plan->threads = kTinyThreads;
        plan->grid = ceil_div(p, (uint64_t)kTinyThreads * kTinyRowsPerThread);
        plan->p = p;
        plan->L = L;
        plan->slots = K;
        plan->U = 1;
        plan->sym_per_lookup = B ? 4 / B : 1;
        plan->win = (policy == PAREM_BOUNDARY_SNAP && L > 1) ? (uint32_t)(L - 1 < 64 ? L - 1 : 64) : 0;
        plan->smem = smem;
        plan->off_maps = 256;
        plan->ws = al256(plan->off_maps + plan->grid * d.Qpad * 8);
        if (plan->grid > 0x7FFFFFFFull) { set_error("too many chunks"); return PAREM_EINVAL; }
        return PAREM_OK;
    }

    if (kernel == kKernelConv) {
        // K2 follows one dependent chain per chunk: the chunk count is the number of
        // lookups in flight (one follow CTA per SM, one wave); the set walk's cost grows with
        // the chunk count, and chunks stay long against the walk's head (~conv_t4 symbols).
        // With the opt-in TMA-staged follow the rows are whole 64-byte boxes (and not
        // multiples of 256 B: TMA row streams at such strides are slower,
        // profiles/r01_stride_probe.txt).
        // L2-resident tables: each thread streams its row with 16-byte loads that do not
        // allocate in L1 (the table keeps the whole L1: carveout 0); the staged follow is
        // slower there (cfg5 18.8 vs 14.2 ms, cfg4 14.0 vs 11.3 ms).
        // Shared-memory tables: the staged follow (rows streamed through shared memory by TMA; 2 =
        // by warp-cooperative cp.async) with the follow table in 8 bank-confined copies
        // (TabR<8>) at 512 chains per SM -- cfg3 follow 1.80 ms against 2.10 ms for the
        // thread-stream follow with the byte-entry table (which stays the fallback when the
        // input is not 16-byte aligned or a chunk length is forced).  The staged follow only
        // became the faster one once the last chunk was kept short (below).
        plan->conv_tma = conv_smem_tab ? 1 : 0;
        plan->set_own = 1;
        if (const char* e = getenv("PAREM_CONV_TMA")) plan->conv_tma = (uint32_t)atoi(e);   // experiments
        // follow table: sixteen byte-entry copies (TabB, 116) when the DFA has <= 256 states and
        // they fit 112 KB -- 2 wavefronts per lookup instead of ~3.6 (cfg3 follow 2.33 -> 2.10
        // ms); else the plain table.  PAREM_CONV_REP = 0 / 8 / 16 / 116 for experiments.
        plan->conv_rep = conv_smem_tab && conv_byte_table_applies(d) ? 116 : 0;
        if (plan->conv_tma && conv_smem_tab) {
            const size_t rb = conv_rep_smem(d, 8);
            if (rb && conv_follow_tma_smem(rb) <= 232448 - 1024) plan->conv_rep = 8;
        }
        if (const char* e = getenv("PAREM_CONV_REP")) plan->conv_rep = (uint32_t)atoi(e);
        if (plan->conv_rep == 116) {   // byte-entry table, 16 copies (TabB)
            if (!conv_smem_tab || !conv_byte_table_applies(d)) plan->conv_rep = 0;
        } else if (plan->conv_rep) {
            const size_t rb = conv_smem_tab ? conv_rep_smem(d, plan->conv_rep) : 0;
            const size_t need = plan->conv_tma ? conv_follow_tma_smem(rb) : rb;
            if (!rb || (plan->conv_rep != 8 && plan->conv_rep != 16) || need > 232448 - 1024) plan->conv_rep = 0;
        }
        if (const char* e = getenv("PAREM_SET_OWN")) plan->set_own = (uint32_t)atoi(e);
        plan->conv_fthreads = 512;
        if (const char* e = getenv("PAREM_CONV_FTHREADS")) plan->conv_fthreads = (uint32_t)atoi(e);   // experiments
        plan->conv_cpt = 1;
        plan->conv_swarps = conv_swarps;
        if (const char* e = getenv("PAREM_CONV_CPT")) plan->conv_cpt = atoi(e) == 2 ? 2 : 1;
        uint64_t L;
        // chains: 512 per SM -- one 512-thread follow CTA per SM, exactly one wave (a partial
        // second wave or unevenly loaded SMs cost more than the extra chains bring); the
        // follow is bound by shared-memory bank conflicts (smem tables) or L1TEX gather
        // wavefronts (L2 tables), not by latency, and more chunks only add set-walk work
        // ... unless the set walk of one chunk (create-time probe: conv_work4 lookups until
        // <= 4 states) costs about as much as following the chunk itself: slowly converging
        // automata (cfg4: ~60 k set-walk lookups against 28 KB chunks) run fewer, longer
        // chunks -- their follow keeps several routes per lane in flight and loses little
        // (cfg4, chains/SM 256 / 320 / 384 / 448 / 512: 22.5 / 21.8 / 23.3 / 24.1 / 26.0 ms per
        // step; cfg5, where the set walk is cheap: 27.4 / 22.9 / 20.1 / 18.4 / 17.3 ms)
        // Hybrid follow table (tables beyond shared memory with <= 1024 states: part of the
        // columns packed in shared memory): faster per lookup but latency-bound at 512
        // chains per SM, so two chunks per thread (1024 chains per SM).  Experimental knob
        // first: PAREM_CONV_HYB=1.
        plan->conv_hyb = 0;
        if (const char* e = getenv("PAREM_CONV_HYB")) plan->conv_hyb = (uint32_t)atoi(e);
        if (plan->conv_hyb && (conv_smem_tab || !conv_hybrid_applies(d) || plan->conv_tma)) plan->conv_hyb = 0;
        if (plan->conv_hyb && !getenv("PAREM_CONV_CPT")) plan->conv_cpt = 2;
        if (!plan->conv_tma && !getenv("PAREM_CONV_FTHREADS")) {
            const double L512 = (double)n / (512.0 * sms);
            const double rho = L512 > 0 ? (double)dfa->conv_work4 / L512 : 0.0;
            plan->conv_fthreads = rho >= 1.5 ? 320 : rho >= 0.75 ? 416 : 512;
        }
        uint64_t chains = (uint64_t)sms * (plan->conv_tma ? 512 : plan->conv_fthreads * plan->conv_cpt);
        uint32_t dmax = 4;
        uint64_t headx = 16;
        if (const char* e = getenv("PAREM_CONV_CHAINS")) chains = strtoull(e, nullptr, 10);   // experiments
        if (const char* e = getenv("PAREM_CONV_HEADX")) headx = strtoull(e, nullptr, 10);
        if (const char* e = getenv("PAREM_CONV_DMAX")) dmax = (uint32_t)atoi(e);
        if ((dmax != 1 && dmax != 2) || dfa->conv_t1 == 0) dmax = 4;
        if (forced) L = forced;
        else {
            L = ceil_div(n, chains ? chains : 1);
            // chunks >= headx times the probe's convergence length, so open chunks (no
            // hand-over, resolved by head walks in the join) stay rare
            const uint64_t head = headx * (dmax == 4 ? dfa->conv_t4 : dfa->conv_t1);
            if (L < head) L = head;
            if (L < 4096) L = 4096;
            if (plan->conv_tma) {
                L = (L + 63) & ~63ull;
                if (L % 256 == 0) L += 64;
                // The last chunk (n mod L bytes, not a full row) is walked by one lane after its
                // warp's staged rows: keep it short -- among the next row lengths take the one
                // with the smallest remainder (a 36 KB last chunk cost cfg3 ~1 ms of 2.9).
                uint64_t bestL = L, bestr = n % L ? n % L : L;
                for (uint64_t c = L; c < L + 64 * 96 && bestr > 2048; c += 64) {
                    if (c % 256 == 0) continue;
                    const uint64_t r = n % c ? n % c : c;
                    if (r < bestr) { bestr = r; bestL = c; }
                }
                L = bestL;
            } else {
                L = (L + 15) & ~15ull;
                // thread-per-chunk 16-B load streams at a stride that is a multiple of 128 B
                // run ~18% slower (profiles/r01_stride_probe.txt): shift such strides by 16 B
                if (L % 128 == 0) L += 16;
            }
        }
        if (L > (1ull << 30)) L = 1ull << 30;
        // planner-chosen lengths: the remainder forms a SHORTER last chunk (p = ceil(n / L)),
        // so no follow thread walks more than L bytes (a forced chunk_len keeps reading C7)
        const uint64_t p = forced ? (n / L ? n / L : 1) : ceil_div(n, L);
        plan->policy = PAREM_BOUNDARY_GRID;   // the converging path uses the paper's partition
        plan->dmax = dmax;
        plan->threads = 512;
        plan->grid = ceil_div(p, 512);
        plan->p = p;
        plan->L = L;
        plan->slots = conv_cap;
        plan->U = 1;
        plan->sym_per_lookup = 1;
        plan->win = 0;
        plan->smem_tab = conv_smem_tab;
        plan->smem = conv_set_smem_bytes(d, conv_smem_tab, conv_cap, conv_swarps);
        plan->off_maps = 256;
        plan->off_hits = 0;
        plan->ws = al256(plan->off_maps + conv_ws_total(p));
        if (p > 0x7FFFFFFFull) { set_error("too many chunks"); return PAREM_EINVAL; }
        return PAREM_OK;
    }

    // lanes
    const size_t ES = d.lanes_u32 ? 4 : 2;
    const size_t tab_bytes = (size_t)d.Apad * d.Qpad * ES;
    const bool smem_tab = tab_bytes <= (size_t)160 * 1024;
    uint32_t S = cand == PAREM_CANDIDATES_ENUM ? d.Q : d.Lmax;
    if (S < 1) S = 1;
    // choose U (routes per thread) and Tg (threads per chunk) minimising the issue cost of
    // one byte: Tg * (3 U + 3) (3 instructions per route-step + ~3 shared per byte)
    static const uint32_t Us[] = {1, 2, 3, 4, 6, 8};
    uint32_t U = 1;
    uint64_t Tg = 32, best = ~0ull;
    for (uint32_t u : Us) {
        uint64_t tg = 32 * ceil_div(S, 32ull * u);
        if (tg > 1024) continue;
        const uint64_t cost = tg * (3ull * u + 3);
        if (cost < best) { best = cost; U = u; Tg = tg; }
    }
    if (best == ~0ull) { U = 8; Tg = 1024; }           // > 8192 candidates: extra passes
    // several chunks per CTA share the staged table: up to 512 threads per CTA
    uint64_t G = Tg >= 512 ? 1 : 512 / Tg;
    if (G > lanes_max_groups()) G = lanes_max_groups();
    const uint64_t T = G * Tg;
    const size_t smem = lanes_smem_bytes(d, smem_tab);
    int bps = cached_bps(2, U, smem_tab, d.lanes_u32, (uint32_t)T, smem);
    if (bps <= 0) { set_error("lanes kernel does not fit (smem %zu, threads %llu)", smem, (unsigned long long)T); return PAREM_EINVAL; }
    uint64_t L;
    if (forced) L = forced;
    else {
        const uint64_t target = (uint64_t)sms * bps * G;   // one wave of chunk groups
        L = ceil_div(n, target);
        L = (L + 15) & ~15ull;
        if (L < 4096) L = 4096;
    }
    if (L > (1ull << 30)) L = 1ull << 30;
    const uint64_t p = n / L ? n / L : 1;
    plan->threads = (uint32_t)T;
    plan->tg = (uint32_t)Tg;
    plan->grid = ceil_div(p, G);
    plan->p = p;
    plan->L = L;
    plan->slots = (uint32_t)(Tg * U);
    plan->U = U;
    plan->sym_per_lookup = 1;
    plan->win = (policy == PAREM_BOUNDARY_SNAP && L > 1) ? (uint32_t)(L - 1 < 4096 ? L - 1 : 4096) : 0;
    plan->smem_tab = smem_tab;
    plan->smem = smem;
    plan->off_maps = 256;
    plan->off_hits = al256(plan->off_maps + p * d.Qpad * 4);
    plan->ws = al256(plan->off_hits + p * d.Qpad * 4);
    if (p > 0x7FFFFFFFull) { set_error("too many chunks"); return PAREM_EINVAL; }
    return PAREM_OK;
}

}  // namespace parem
