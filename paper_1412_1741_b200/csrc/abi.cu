// abi.cu -- the C ABI entry points (include/parem.h): planning, workspace sizing, the
// async / sync / continue / host-buffer match calls, and the roofline micro-benchmarks.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only; a no-op unless a tool (nsys, ncu --nvtx) is attached

#include "kernels_common.cuh"

namespace parem {

// n = 0: the result is (q0, q0 in F, 0) (reading C12), composed with the carry.
__global__ void trivial_kernel(const MatchParams P) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        bool dead;
        const uint32_t q = start_state(P, &dead);
        write_result(P, q, 0ull, dead);
    }
}

int launch_trivial(const MatchParams& P, cudaStream_t s) {
    trivial_kernel<<<1, 32, 0, s>>>(P);
    prof_after("trivial", s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("trivial kernel: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    return PAREM_OK;
}

// ---- per-kernel timing (parem_profile) ----
namespace {
struct ProfRec {
    cudaEvent_t start, stop;
    std::string name;
    uint32_t match;
};
struct ProfState {
    bool on = false;
    bool active = false;        // the current match records events
    cudaEvent_t last = nullptr; // event after the previous kernel of the current match
    uint32_t matches = 0;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<ProfRec> recs;
};
thread_local ProfState g_prof;

cudaEvent_t prof_event() {
    ProfState& p = g_prof;
    if (p.used == p.pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        p.pool.push_back(e);
    }
    return p.pool[p.used++];
}

void prof_begin(cudaStream_t s) {
    ProfState& p = g_prof;
    p.active = false;
    if (!p.on) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    cudaEvent_t e = prof_event();
    if (!e) return;
    cudaEventRecord(e, s);
    p.last = e;
    p.active = true;
    ++p.matches;
}
}  // namespace

cudaError_t smem_optin(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> cur;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    size_t& have = cur[{fn, dev}];
    if (bytes <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

void prof_after(const char* name, cudaStream_t s) {
    ProfState& p = g_prof;
    if (!p.active) return;
    cudaEvent_t e = prof_event();
    if (!e) return;
    cudaEventRecord(e, s);
    p.recs.push_back(ProfRec{p.last, e, name, p.matches - 1});
    p.last = e;
}

// NVTX range over the host side of one ABI call (tracing)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

static int match_impl(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, uint64_t offset_base, void* d_ws,
                      size_t ws_bytes, const parem_options* opts, const parem_result* d_carry,
                      parem_result* d_result, cudaStream_t stream, uint64_t* d_positions = nullptr,
                      uint64_t max_positions = 0, bool find = false, uint32_t* d_trace = nullptr, uint64_t tlo = 0,
                      uint64_t thi = 0) {
    set_error("");
    if (!dfa || !d_result) { set_error("null dfa or result"); return PAREM_EINVAL; }
    if (n > 0 && !d_input) { set_error("null input"); return PAREM_EINVAL; }
    Plan plan;
    int rc = make_plan(dfa, n, opts, &plan);
    if (rc != PAREM_OK) return rc;
    if (!d_ws || (reinterpret_cast<uintptr_t>(d_ws) & 15)) { set_error("null or unaligned (16 B) workspace"); return PAREM_EINVAL; }
    if (d_result && (reinterpret_cast<uintptr_t>(d_result) & 7)) { set_error("result must be 8-byte aligned"); return PAREM_EINVAL; }
    const size_t need = find ? ((plan.ws + 255) & ~(size_t)255) + find_extra_bytes(plan, dfa->dev) : plan.ws;
    if (ws_bytes < need) {
        set_error("workspace too small: %zu < %zu", ws_bytes, need);
        return PAREM_ENOMEM;
    }
    if (find && max_positions && !d_positions) {
        set_error("null positions buffer");
        return PAREM_EINVAL;
    }
    MatchParams P;
    memset(&P, 0, sizeof(P));
    P.d = dfa->dev;
    P.in = d_input;
    P.n = n;
    P.L = plan.L;
    P.p = plan.p;
    P.policy = plan.policy;
    P.cand = plan.cand;
    P.win = plan.win;
    P.slots = plan.slots;
    P.tg = plan.tg;
    P.dmax = plan.dmax;
    P.conv_cpt = plan.conv_cpt;
    P.set_own = plan.set_own;
    P.lookback = opts ? opts->lookback : 0;
    P.offset_base = offset_base;
    P.carry = d_carry;
    P.result = d_result;
    P.hdr = reinterpret_cast<WsHeader*>(d_ws);
    P.maps = reinterpret_cast<char*>(d_ws) + plan.off_maps;
    P.map_hits = plan.off_hits ? reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(d_ws) + plan.off_hits) : nullptr;
    if (!(opts && (opts->flags & PAREM_FLAG_WS_CLEAN))) {
        cudaError_t e = cudaMemsetAsync(d_ws, 0, sizeof(WsHeader), stream);
        if (e != cudaSuccess) {
            set_error("cudaMemsetAsync: %s", cudaGetErrorString(e));
            return PAREM_ECUDA;
        }
    }
    prof_begin(stream);
    static const char* const kRangeNames[2][4] = {
        {"parem_match:trivial", "parem_match:tiny", "parem_match:lanes", "parem_match:conv"},
        {"parem_find:trivial", "parem_find:tiny", "parem_find:lanes", "parem_find:conv"}};
    NvtxRange range(kRangeNames[find ? 1 : 0][plan.kernel & 3u]);
    if (plan.kernel == kKernelTrivial) return launch_trivial(P, stream);
    if (find) {
        find_bind(plan, P, reinterpret_cast<unsigned char*>(d_ws) + ((plan.ws + 255) & ~(size_t)255));
        P.fout = d_positions;
        P.fmax = d_positions ? max_positions : 0;
        P.tout = d_trace;
        P.tlo = tlo;
        P.thi = thi;
        if (plan.kernel != kKernelTiny) P.fmend = nullptr;   // only the tiny kernel keeps dense maps
    }
    int rc2;
    if (plan.kernel == kKernelTiny) rc2 = launch_tiny(plan, P, stream);
    else if (plan.kernel == kKernelConv) rc2 = launch_conv(plan, P, stream);
    else rc2 = launch_lanes(plan, P, stream);
    if (rc2 != PAREM_OK || !find) return rc2;
    return launch_find(plan, P, stream);
}

}  // namespace parem

using namespace parem;

extern "C" size_t parem_workspace_bytes(const parem_dfa* dfa, uint64_t n, const parem_options* opts) {
    Plan plan;
    if (make_plan(dfa, n, opts, &plan) != PAREM_OK) return 0;
    return plan.ws;
}

extern "C" int parem_plan(const parem_dfa* dfa, uint64_t n, const parem_options* opts, parem_plan_info* out) {
    if (!out) { set_error("null out"); return PAREM_EINVAL; }
    Plan plan;
    int rc = make_plan(dfa, n, opts, &plan);
    if (rc != PAREM_OK) return rc;
    memset(out, 0, sizeof(*out));
    out->kernel = plan.kernel;
    out->block_threads = plan.threads;
    out->grid_blocks = plan.grid;
    out->num_chunks = plan.p;
    out->chunk_len = plan.L;
    out->boundary_policy = plan.policy;
    out->candidates = plan.cand;
    out->slots = plan.slots;
    out->symbols_per_lookup = plan.sym_per_lookup;
    out->smem_bytes = plan.smem;
    out->workspace_bytes = plan.ws;
    out->snap_window = plan.win;
    return PAREM_OK;
}

extern "C" int parem_match_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, void* d_ws, size_t ws_bytes,
                                 const parem_options* opts, parem_result* d_result, void* stream) {
    return match_impl(dfa, d_input, n, 0, d_ws, ws_bytes, opts, nullptr, d_result, (cudaStream_t)stream);
}

// ---- batched matching: many independent inputs in one launch (tiny kernel) ----
namespace parem {
namespace {
// Batch plan: the tiny kernel with every input an exact multiple of its 1024-chunk CTA tile
// (chunk length a multiple of the 64-byte TMA box), so no warp or CTA spans two inputs.
// Returns false if the batch cannot run as one launch (the caller loops over the inputs).
bool batch_plan(const parem_dfa* dfa, uint64_t n, uint64_t count, const parem_options* opts, Plan* plan,
                uint64_t* cpi) {
    if (!dfa || n == 0 || count == 0) return false;
    if (opts && (opts->candidates == PAREM_CANDIDATES_LOOKBACK || opts->boundary_policy == PAREM_BOUNDARY_SNAP ||
                 (opts->kernel && opts->kernel != kKernelTiny)))
        return false;
    if (make_plan(dfa, n, opts, plan) != PAREM_OK || plan->kernel != kKernelTiny || !plan->tma) return false;
    const uint64_t rows = (uint64_t)kTinyThreads * kTinyRowsPerThread;   // chunks per CTA tile
    const int sms = dfa->num_sms > 0 ? dfa->num_sms : 148;
    // Chunks per input cpi = n / L: whole CTA tiles (cpi a multiple of `rows`), or -- short
    // inputs -- a whole number of warps with several inputs per tile (cpi = 64 .. rows / 2, a
    // power of two), so that 1 MiB inputs still get 4 KiB chunks instead of 512 B ones.
    // Cost: waves x (boxes per row + ~10 box-times of fixed cost per CTA wave; measured on
    // 508 x 1 MiB: 512-byte chunks in 7 waves ran at 2.46 TB/s, 17 us of 31 us per wave fixed).
    uint64_t bestL = 0, best = ~0ull;
    const uint64_t warp_rows = 32ull * kTinyRowsPerThread;
    for (uint64_t L = 64; L <= 16384; L *= 2) {
        if (opts && opts->chunk_len && opts->chunk_len != L) continue;
        if (n % L) continue;
        const uint64_t c = n / L;
        const bool whole = c % rows == 0;
        const bool sub = c >= warp_rows && c < rows && rows % c == 0;
        if (!whole && !sub) continue;
        const uint64_t ctas = (count * c + rows - 1) / rows;
        const uint64_t waves = (ctas + sms - 1) / sms;
        const uint64_t cost = waves * (L / 64 + 10);
        if (cost < best) { best = cost; bestL = L; }
    }
    if (!bestL) return false;
    *cpi = n / bestL;
    const uint64_t ctas = (count * *cpi + rows - 1) / rows;
    if (ctas > 0x7FFFFFFFull) return false;
    const uint64_t spt = *cpi < rows ? rows / *cpi : 1;   // inputs (maps) per CTA tile
    plan->L = bestL;
    plan->p = count * *cpi;
    plan->grid = ctas;
    plan->policy = PAREM_BOUNDARY_GRID;
    plan->win = 0;
    plan->off_maps = 256 + ((count * 32 + 255) & ~255ull);
    plan->ws = ((plan->off_maps + ctas * spt * dfa->dev.Qpad * 8) + 255) & ~(size_t)255;
    return true;
}
}  // namespace
}  // namespace parem

extern "C" size_t parem_batch_workspace_bytes(const parem_dfa* dfa, uint64_t n, uint64_t count,
                                              const parem_options* opts) {
    Plan plan;
    uint64_t cpi = 0;
    const size_t one = parem_workspace_bytes(dfa, n, opts);
    if (!one) return 0;
    if (batch_plan(dfa, n, count, opts, &plan, &cpi)) return plan.ws > one ? plan.ws : one;
    return one;
}

extern "C" int parem_match_batch_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, uint64_t count,
                                       void* d_ws, size_t ws_bytes, const parem_options* opts,
                                       parem_result* d_results, void* stream_) {
    NvtxRange nvtx_range("parem_match_batch");
    set_error("");
    cudaStream_t stream = (cudaStream_t)stream_;
    if (!dfa || !d_results || (count && n && !d_input)) { set_error("null argument"); return PAREM_EINVAL; }
    if (count == 0) return PAREM_OK;
    if (!d_ws || (reinterpret_cast<uintptr_t>(d_ws) & 15)) { set_error("null or unaligned (16 B) workspace"); return PAREM_EINVAL; }
    if (reinterpret_cast<uintptr_t>(d_results) & 7) { set_error("results must be 8-byte aligned"); return PAREM_EINVAL; }
    Plan plan;
    uint64_t cpi = 0;
    if (!(((uintptr_t)d_input) & 15) && batch_plan(dfa, n, count, opts, &plan, &cpi)) {
        if (ws_bytes < plan.ws) { set_error("workspace too small: %zu < %zu", ws_bytes, plan.ws); return PAREM_ENOMEM; }
        MatchParams P;
        memset(&P, 0, sizeof(P));
        P.d = dfa->dev;
        P.in = d_input;
        P.n = n * count;
        P.L = plan.L;
        P.p = plan.p;
        P.policy = PAREM_BOUNDARY_GRID;
        P.cand = plan.cand;
        P.slots = plan.slots;
        P.hdr = reinterpret_cast<WsHeader*>(d_ws);
        P.bstats = reinterpret_cast<unsigned long long*>(static_cast<char*>(d_ws) + 256);
        P.maps = static_cast<char*>(d_ws) + plan.off_maps;
        P.cpi = cpi;
        P.n_one = n;
        P.results = d_results;
        if (!(opts && (opts->flags & PAREM_FLAG_WS_CLEAN))) {
            cudaError_t e = cudaMemsetAsync(d_ws, 0, plan.off_maps, stream);
            if (e != cudaSuccess) { set_error("cudaMemsetAsync: %s", cudaGetErrorString(e)); return PAREM_ECUDA; }
        }
        prof_begin(stream);
        return launch_tiny(plan, P, stream);
    }
    // general case: one match per input, in order on the stream (they share the workspace)
    for (uint64_t i = 0; i < count; ++i) {
        const int rc = match_impl(dfa, d_input + i * n, n, 0, d_ws, ws_bytes, opts, nullptr, d_results + i, stream);
        if (rc != PAREM_OK) return rc;
    }
    return PAREM_OK;
}

// ---- sharding one input over GPUs: segment maps and their fold ----
extern "C" int parem_segment_map(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, int32_t prev_symbol,
                                 const parem_options* opts, parem_segmap_entry* h_map, int32_t* status,
                                 uint64_t* bad_offset, void* stream_) {
    NvtxRange nvtx_range("parem_segment_map");
    set_error("");
    if (!dfa || !h_map || !status || !bad_offset || (n && !d_input)) { set_error("null argument"); return PAREM_EINVAL; }
    cudaStream_t stream = (cudaStream_t)stream_;
    const DevDfa& d = dfa->dev;
    const uint32_t Q = dfa->Q;
    for (uint32_t q = 0; q < Q; ++q) h_map[q] = parem_segmap_entry{0, 0, 0};
    *status = PAREM_OK;
    *bad_offset = 0;
    // candidates R: {q0} for the first segment, else L(prev) (all of Q after an invalid byte:
    // the previous segment reports that ESYMBOL)
    uint32_t loff = 0, ncand = 1;
    const bool first = prev_symbol < 0;
    if (!first) {
        const uint32_t li = (uint32_t)prev_symbol < dfa->A ? (uint32_t)prev_symbol : dfa->A;
        cudaError_t e = cudaMemcpy(&loff, d.Loff + li, 4, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(&ncand, d.Lcnt + li, 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { set_error("segment map: %s", cudaGetErrorString(e)); return PAREM_ECUDA; }
    }
    // R empty (C10): nothing enters this segment alive -- the map stays invalid, but every
    // byte is still validated (C11): one placeholder walker covers the whole segment
    const bool empty = ncand == 0;
    if (empty) ncand = 1;
    std::vector<uint32_t> cand(ncand);
    if (first || empty) cand[0] = first ? dfa->start : 0u;
    else if (ncand && cudaMemcpy(cand.data(), d.Llist + loff, 4ull * ncand, cudaMemcpyDeviceToHost) != cudaSuccess) {
        set_error("segment map: candidate copy failed");
        return PAREM_ECUDA;
    }
    if (n == 0) {
        if (!empty)
            for (uint32_t r : cand) h_map[r] = parem_segmap_entry{0, r, 1};
        return PAREM_OK;
    }
    // device scratch: candidates, head states, head hits, bad offset, carry + result
    const size_t c4 = (4ull * ncand + 255) & ~255ull, c8 = (8ull * ncand + 255) & ~255ull;
    void* blk = nullptr;
    cudaError_t e = cudaMalloc(&blk, 2 * c4 + c8 + 512);
    if (e != cudaSuccess) { set_error("cudaMalloc: %s", cudaGetErrorString(e)); return PAREM_ENOMEM; }
    uint32_t* d_cand = static_cast<uint32_t*>(blk);
    uint32_t* d_st = reinterpret_cast<uint32_t*>(static_cast<char*>(blk) + c4);
    unsigned long long* d_hits = reinterpret_cast<unsigned long long*>(static_cast<char*>(blk) + 2 * c4);
    unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(static_cast<char*>(blk) + 2 * c4 + c8);
    parem_result* d_res = reinterpret_cast<parem_result*>(static_cast<char*>(blk) + 2 * c4 + c8 + 256);
    int rc = PAREM_OK;
    std::vector<uint32_t> st(ncand);
    std::vector<unsigned long long> hits(ncand);
    unsigned long long bad_inv = 0;
    // head length: a multiple of the create-time convergence probe, grown until the heads
    // end in <= 32 distinct states (or cover the whole segment)
    const uint64_t conv = dfa->conv_t1 ? dfa->conv_t1 : (dfa->conv_t4 ? 4ull * dfa->conv_t4 : 1024);
    uint64_t X = empty ? n : std::min<uint64_t>(n, std::max<uint64_t>(4096, 4 * conv));
    std::vector<uint32_t> zs;
    e = cudaMemcpyAsync(d_cand, cand.data(), 4ull * ncand, cudaMemcpyHostToDevice, stream);
    for (;;) {
        if (e == cudaSuccess) e = cudaMemsetAsync(d_bad, 0, 8, stream);
        if (e != cudaSuccess) { set_error("segment map: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; break; }
        rc = launch_segment_head(d, d_input, X, d_cand, ncand, d_st, d_hits, d_bad, stream);
        if (rc != PAREM_OK) break;
        e = cudaMemcpyAsync(st.data(), d_st, 4ull * ncand, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hits.data(), d_hits, 8ull * ncand, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&bad_inv, d_bad, 8, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) { set_error("segment map: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; break; }
        zs.assign(st.begin(), st.end());
        std::sort(zs.begin(), zs.end());
        zs.erase(std::unique(zs.begin(), zs.end()), zs.end());
        if (zs.size() <= 32 || X == n) break;
        X = std::min<uint64_t>(n, 4 * X);
    }
    // finish every distinct head state over [X, n) with one ordinary match
    std::vector<uint32_t> zend(zs.size());
    std::vector<uint64_t> zcnt(zs.size(), 0);
    if (rc == PAREM_OK && X < n) {
        const size_t ws = parem_workspace_bytes(dfa, n - X, opts);
        void* d_ws = nullptr;
        if (!ws || cudaMalloc(&d_ws, ws) != cudaSuccess) { set_error("segment map: workspace"); rc = PAREM_ENOMEM; }
        for (size_t j = 0; rc == PAREM_OK && j < zs.size(); ++j) {
            parem_result carry;
            memset(&carry, 0, sizeof(carry));
            carry.final_state = zs[j] == d.sink && d.has_sink ? PAREM_DEAD : zs[j];
            parem_result r;
            e = cudaMemcpyAsync(d_res, &carry, sizeof(carry), cudaMemcpyHostToDevice, stream);
            if (e == cudaSuccess) e = cudaMemsetAsync(d_ws, 0, 64, stream);
            if (e != cudaSuccess) { set_error("segment map: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; break; }
            rc = match_impl(dfa, d_input + X, n - X, X, d_ws, ws, opts, d_res, d_res, stream);
            if (rc != PAREM_OK) break;
            e = cudaMemcpyAsync(&r, d_res, sizeof(r), cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
            if (e != cudaSuccess) { set_error("segment map: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; break; }
            if (r.status == PAREM_ESYMBOL) {
                *status = PAREM_ESYMBOL;
                *bad_offset = r.bad_offset;   // offset_base X: local to the segment
            } else if (r.status != PAREM_OK) {
                rc = r.status;
                break;
            }
            zend[j] = r.final_state;
            zcnt[j] = r.match_count;
        }
        if (d_ws) cudaFree(d_ws);
    }
    cudaFree(blk);
    if (rc != PAREM_OK) return rc;
    if (bad_inv) {   // an invalid byte inside the head comes first
        *status = PAREM_ESYMBOL;
        *bad_offset = ~bad_inv;
    }
    for (uint32_t i = 0; i < ncand && !empty; ++i) {
        const size_t j = std::lower_bound(zs.begin(), zs.end(), st[i]) - zs.begin();
        uint32_t end = X < n ? zend[j] : st[i];
        if (X == n && d.has_sink && end == d.sink) end = PAREM_DEAD;
        h_map[cand[i]] = parem_segmap_entry{hits[i] + (X < n ? zcnt[j] : 0ull), end, 1u};
    }
    return PAREM_OK;
}

extern "C" int parem_fold_segment_maps(uint32_t Q, uint32_t q0, const uint8_t* accept_bitmap,
                                       const parem_segmap_entry* maps, uint32_t G, const int32_t* statuses,
                                       const uint64_t* bad_offsets, const uint64_t* seg_offsets, parem_result* out) {
    if (!out || !accept_bitmap || (G && (!maps || !statuses || !bad_offsets || !seg_offsets)) || q0 >= Q) {
        set_error("null argument");
        return PAREM_EINVAL;
    }
    parem_result r;
    memset(&r, 0, sizeof(r));
    r.num_chunks = G;
    uint32_t q = q0;
    uint64_t count = 0;
    for (uint32_t g = 0; g < G; ++g) {
        if (statuses[g] == PAREM_ESYMBOL && r.status != PAREM_ESYMBOL) {
            r.status = PAREM_ESYMBOL;
            r.bad_offset = seg_offsets[g] + bad_offsets[g];
        }
        if (q == PAREM_DEAD) continue;   // a dead walk stays dead (reading C9)
        const parem_segmap_entry& e = maps[(uint64_t)g * Q + q];
        if (!e.valid) {
            set_error("segment %u entered in state %u, not one of its candidates", g, q);
            return PAREM_EINTERNAL;
        }
        count += e.match_count;
        q = e.end_state;
    }
    r.final_state = q;
    r.accepted = q != PAREM_DEAD && ((accept_bitmap[q >> 3] >> (q & 7)) & 1);
    r.match_count = count;
    *out = r;
    return r.status;
}

extern "C" int parem_match_continue_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n,
                                          uint64_t offset_base, void* d_ws, size_t ws_bytes,
                                          const parem_options* opts, const parem_result* d_carry,
                                          parem_result* d_result, void* stream) {
    return match_impl(dfa, d_input, n, offset_base, d_ws, ws_bytes, opts, d_carry, d_result, (cudaStream_t)stream);
}

extern "C" int parem_match(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, const parem_options* opts,
                           parem_result* h_result, void* stream_) {
    if (!h_result) { set_error("null result"); return PAREM_EINVAL; }
    cudaStream_t stream = (cudaStream_t)stream_;
    const size_t ws = parem_workspace_bytes(dfa, n, opts);
    if (!ws) return PAREM_EINVAL;
    void* blk = nullptr;
    const size_t ws_al = (ws + 255) & ~(size_t)255;
    cudaError_t e = cudaMallocAsync(&blk, ws_al + 256, stream);
    if (e != cudaSuccess) { set_error("cudaMallocAsync: %s", cudaGetErrorString(e)); return PAREM_ENOMEM; }
    parem_result* d_res = reinterpret_cast<parem_result*>(static_cast<char*>(blk) + ws_al);
    int rc = match_impl(dfa, d_input, n, 0, blk, ws, opts, nullptr, d_res, stream);
    if (rc == PAREM_OK) {
        e = cudaMemcpyAsync(h_result, d_res, sizeof(parem_result), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) { set_error("match: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; }
    }
    cudaFreeAsync(blk, stream);
    if (rc != PAREM_OK) return rc;
    return h_result->status;
}

// Per-thread, per-device resources of parem_match_host: the copy stream and its events are
// created once and reused (creating a stream and five events per call cost more than a
// small match).  Deliberately never destroyed (process lifetime; the driver reclaims them).
namespace parem {
namespace {
struct HostPipe {
    int dev = -1;
    cudaStream_t cs = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr}, ready = nullptr;
};
cudaError_t host_pipe(HostPipe** out) {
    static thread_local HostPipe pipes[8];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    HostPipe& h = pipes[dev & 7];
    if (h.dev != dev) {
        e = cudaStreamCreateWithFlags(&h.cs, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&h.copied[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.used[i], cudaEventDisableTiming);
        }
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.ready, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
        h.dev = dev;
    }
    *out = &h;
    return cudaSuccess;
}
}  // namespace
}  // namespace parem

extern "C" int parem_match_host(const parem_dfa* dfa, const uint8_t* h_input, uint64_t n, const parem_options* opts,
                                parem_result* h_result, void* stream_) {
    NvtxRange nvtx_range("parem_match_host");
    if (!h_result || !dfa || (n && !h_input)) { set_error("null argument"); return PAREM_EINVAL; }
    cudaStream_t stream = (cudaStream_t)stream_;
    // segments: 64 MiB for the tiny kernel; 512 MiB for the large-DFA paths, whose per-match
    // cost has a part that scales with the chunk count rather than the bytes
    Plan probe;
    uint64_t SEG = 64ull << 20;
    if (n > SEG && make_plan(dfa, SEG, opts, &probe) == PAREM_OK && probe.kernel != kKernelTiny) SEG = 512ull << 20;
    const uint64_t seg = n < SEG ? (n ? n : 1) : SEG;
    const size_t ws = parem_workspace_bytes(dfa, seg, opts);
    if (!ws) return PAREM_EINVAL;
    const size_t seg_al = (seg + 255) & ~(size_t)255, ws_al = (ws + 255) & ~(size_t)255;
    const size_t bytes = 2 * seg_al + ws_al + 256;
    HostPipe* hp = nullptr;
    cudaError_t e = host_pipe(&hp);
    if (e != cudaSuccess) { set_error("stream setup: %s", cudaGetErrorString(e)); return PAREM_ECUDA; }
    void* blk = nullptr;
    e = cudaMallocAsync(&blk, bytes, stream);
    if (e != cudaSuccess) { set_error("cudaMallocAsync: %s", cudaGetErrorString(e)); return PAREM_ENOMEM; }
    uint8_t* buf[2] = {static_cast<uint8_t*>(blk), static_cast<uint8_t*>(blk) + seg_al};
    void* d_ws = static_cast<uint8_t*>(blk) + 2 * seg_al;
    parem_result* d_res = reinterpret_cast<parem_result*>(static_cast<uint8_t*>(blk) + 2 * seg_al + ws_al);
    cudaStream_t cs = hp->cs;
    int rc = PAREM_OK;
    // the copy stream must not start before the buffers exist on `stream`
    e = cudaEventRecord(hp->ready, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, hp->ready, 0);
    if (e != cudaSuccess) {
        set_error("stream setup: %s", cudaGetErrorString(e));
        rc = PAREM_ECUDA;
    }
    if (rc == PAREM_OK && n == 0) rc = match_impl(dfa, nullptr, 0, 0, d_ws, ws, opts, nullptr, d_res, stream);
    uint64_t k = 0;
    for (uint64_t off = 0; rc == PAREM_OK && off < n; off += seg, ++k) {
        const uint64_t len = n - off < seg ? n - off : seg;
        const int b = (int)(k & 1);
        if (k >= 2) cudaStreamWaitEvent(cs, hp->used[b], 0);
        e = cudaMemcpyAsync(buf[b], h_input + off, len, cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess) e = cudaEventRecord(hp->copied[b], cs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, hp->copied[b], 0);
        if (e != cudaSuccess) { set_error("H2D: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; break; }
        rc = match_impl(dfa, buf[b], len, off, d_ws, ws, opts, off ? d_res : nullptr, d_res, stream);
        if (rc == PAREM_OK && cudaEventRecord(hp->used[b], stream) != cudaSuccess) rc = PAREM_ECUDA;
    }
    if (rc == PAREM_OK) {
        e = cudaMemcpyAsync(h_result, d_res, sizeof(parem_result), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) { set_error("match_host: %s", cudaGetErrorString(e)); rc = PAREM_ECUDA; }
    } else {
        cudaStreamSynchronize(stream);
    }
    cudaStreamSynchronize(cs);
    cudaFreeAsync(blk, stream);
    if (rc != PAREM_OK) return rc;
    return h_result->status;
}

// ------------------------------------------------------------------------------------
// Roofline micro-benchmarks (bench.py measures the denominators in the same run).
// ------------------------------------------------------------------------------------
namespace parem {

__global__ void __launch_bounds__(512) read_stream_kernel(const uint4* __restrict__ in, uint64_t nvec,
                                                          uint32_t* sink) {
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nvec; i += 4 * stride) {
        uint4 a = ldg_v4(reinterpret_cast<const uint8_t*>(in + i));
        uint4 b = ldg_v4(reinterpret_cast<const uint8_t*>(in + i + stride));
        uint4 c = ldg_v4(reinterpret_cast<const uint8_t*>(in + i + 2 * stride));
        uint4 d = ldg_v4(reinterpret_cast<const uint8_t*>(in + i + 3 * stride));
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    for (; i < nvec; i += stride) {
        uint4 a = ldg_v4(reinterpret_cast<const uint8_t*>(in + i));
        acc ^= a.x ^ a.y ^ a.z ^ a.w;
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;   // practically never; keeps the loads alive
}

// Dependent random gathers, 8 independent chains per thread, `steps` steps each, so the
// LSU (not the chain latency) is the limit at full occupancy.
// where = 0: u32 table in shared memory (random banks, the lanes kernel's access pattern);
//         1: u16 table in global memory / L2;
//         2: u32 table in shared memory, lane-private (word w of lane l at w*32 + l:
//            conflict-free by construction -- the tiny kernel's stride-table pattern).
template <int WHERE>
__global__ void __launch_bounds__(256) gather_kernel(const uint16_t* __restrict__ tab, uint32_t entries,
                                                     uint32_t steps, uint32_t* sink) {
    extern __shared__ __align__(16) unsigned char smb[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const uint32_t mask = entries - 1u;   // entries is a power of two
    uint32_t* t32 = reinterpret_cast<uint32_t*>(smb);
    if (WHERE == 0)
        for (uint32_t i = tid; i < entries; i += blockDim.x) t32[i] = tab[i];
    if (WHERE == 2)
        for (uint32_t i = tid; i < entries * 32u; i += blockDim.x) t32[i] = tab[i >> 5];
    __syncthreads();
    uint32_t x[8], rng[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = (blockIdx.x * 977u + tid * 131u + 37u * k) & mask;
        rng[k] = (blockIdx.x * blockDim.x + tid) * 747796405u + 2891336453u * (uint32_t)(k + 1);
    }
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t v;
            if (WHERE == 0) v = t32[x[k]];
            else if (WHERE == 1) v = __ldg(tab + x[k]);
            else v = t32[x[k] * 32u + lane];
            // Next index = loaded value (the "state") + this chain's OWN pseudo-random stream
            // (the "symbol"), scattered over the whole table.  Round 2's first version added
            // the step number instead: every chain then applied the SAME map per step, so
            // chains that met stayed together (the route merging of the paper, in
            // the benchmark itself), lanes shared addresses and the rate was overstated ~2x
            // (profiles/r02_follow_probe.txt).
            // Lane-private tables (WHERE == 2) cannot share addresses between chains, so they
            // keep the cheap index update: the added arithmetic would make that probe
            // issue-bound instead of shared-memory-bound.
            if (WHERE == 2) {
                x[k] = (v * 0x9E3779B1u + s) & mask;
            } else {
                rng[k] = rng[k] * 1664525u + 1013904223u;
                x[k] = ((v + (rng[k] >> 8)) * 0x9E3779B1u >> 7) & mask;
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= x[k];
    if (acc == sink[1]) sink[0] = acc;   // the caller's sink[1] is never a reachable value
}

}  // namespace parem

extern "C" size_t parem_find_workspace_bytes(const parem_dfa* dfa, uint64_t n, const parem_options* opts) {
    Plan plan;
    if (make_plan(dfa, n, opts, &plan) != PAREM_OK) return 0;
    if (plan.kernel == kKernelTrivial) return plan.ws;
    return ((plan.ws + 255) & ~(size_t)255) + find_extra_bytes(plan, dfa->dev);
}

extern "C" int parem_find_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, void* d_ws, size_t ws_bytes,
                                const parem_options* opts, uint64_t* d_positions, uint64_t max_positions,
                                parem_result* d_result, void* stream) {
    return match_impl(dfa, d_input, n, 0, d_ws, ws_bytes, opts, nullptr, d_result, (cudaStream_t)stream, d_positions,
                      max_positions, true);
}

extern "C" int parem_trace_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, void* d_ws, size_t ws_bytes,
                                 const parem_options* opts, uint64_t lo, uint64_t hi, uint32_t* d_states,
                                 parem_result* d_result, void* stream) {
    if (lo > hi || hi > n) {
        set_error("trace window [%llu, %llu) outside the input (n = %llu)", (unsigned long long)lo,
                  (unsigned long long)hi, (unsigned long long)n);
        return PAREM_EINVAL;
    }
    if (hi > lo && !d_states) {
        set_error("null trace buffer");
        return PAREM_EINVAL;
    }
    return match_impl(dfa, d_input, n, 0, d_ws, ws_bytes, opts, nullptr, d_result, (cudaStream_t)stream, nullptr, 0, true,
                      d_states, lo, hi);
}

extern "C" int parem_profile(int enable) {
    ProfState& p = g_prof;
    if (enable) {
        p.used = 0;
        p.recs.clear();
        p.matches = 0;
    }
    p.on = enable != 0;
    p.active = false;
    return PAREM_OK;
}

extern "C" int parem_profile_read(parem_kernel_time* out, int max, int* count) {
    ProfState& p = g_prof;
    const int nk = (int)p.recs.size();
    if (count) *count = nk;
    for (int k = 0; k < nk && k < max; ++k) {
        const ProfRec& r = p.recs[k];
        if (cudaEventSynchronize(r.stop) != cudaSuccess) {
            set_error("parem_profile_read: event sync failed");
            return PAREM_ECUDA;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, r.start, r.stop);
        memset(out[k].name, 0, sizeof(out[k].name));
        strncpy(out[k].name, r.name.c_str(), sizeof(out[k].name) - 1);
        out[k].ms = ms;
        out[k].match = r.match;
    }
    return PAREM_OK;
}

extern "C" float parem_bench_read_stream(const uint8_t* d_input, uint64_t n, uint32_t* d_sink, int reps,
                                         void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (!d_input || (((uintptr_t)d_input) & 15) || reps < 1) return (float)PAREM_EINVAL;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint64_t nvec = n / 16;
    read_stream_kernel<<<sms * 4, 512, 0, stream>>>(reinterpret_cast<const uint4*>(d_input), nvec, d_sink);
    cudaEventRecord(a, stream);
    for (int r = 0; r < reps; ++r)
        read_stream_kernel<<<sms * 4, 512, 0, stream>>>(reinterpret_cast<const uint4*>(d_input), nvec, d_sink);
    cudaEventRecord(b, stream);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (cudaGetLastError() != cudaSuccess) return (float)PAREM_ECUDA;
    return ms / reps;
}

extern "C" float parem_bench_gather(uint32_t where, const uint16_t* d_table, uint32_t entries, uint32_t steps,
                                    uint32_t* d_sink, uint64_t* lookups_out, int reps, void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (!d_table || entries == 0 || (entries & (entries - 1)) || reps < 1 || where > 2) return (float)PAREM_EINVAL;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t smem = where == 0 ? (size_t)entries * 4 : where == 2 ? (size_t)entries * 128 : 0;
    if (smem > 200 * 1024) return (float)PAREM_EINVAL;
    const void* fn = where == 0 ? (const void*)gather_kernel<0> : where == 1 ? (const void*)gather_kernel<1>
                                                                           : (const void*)gather_kernel<2>;
    smem_optin(fn, smem);
    int bps = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, 256, smem);
    if (bps < 1) bps = 1;
    const unsigned grid = (unsigned)(sms * bps);
    void* args[] = {(void*)&d_table, (void*)&entries, (void*)&steps, (void*)&d_sink};
    cudaLaunchKernel(fn, dim3(grid), dim3(256), args, smem, stream);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, stream);
    for (int r = 0; r < reps; ++r) cudaLaunchKernel(fn, dim3(grid), dim3(256), args, smem, stream);
    cudaEventRecord(b, stream);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (lookups_out) *lookups_out = (uint64_t)grid * 256 * 8 * steps;
    if (cudaGetLastError() != cudaSuccess) return (float)PAREM_ECUDA;
    return ms / reps;
}
