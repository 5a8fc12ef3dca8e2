// kernels_tiny.cu -- multi-start chunk simulation for small DFAs (internal states <= 32):
// one THREAD per chunk, the chunk's candidate start states R_i as K registers that all
// advance in one pass over the chunk's bytes (Alg. 1 lines 16-25), dense
// per-chunk maps start -> (end, hits) composed by warps, and a
// last-CTA fold of the per-CTA tile maps along q0's path.
//
// Input staging (TMA variant): chunk t is row t of a 2-D tensor view of the input (row
// length = nominal chunk length L); each warp streams its 32 rows through shared memory in
// 32 x 64-byte boxes with cp.async.bulk.tensor (SWIZZLE_64B, so the 8 lanes of an LDS.128
// phase hit distinct banks), double-buffered on mbarriers.  Without TMA (unaligned input,
// forced odd chunk lengths) each lane streams its own chunk with 16-byte loads.
//
// Lookup tables in shared memory:
//   * A <= 4: a 4-bit-group STRIDE table; one lookup advances a route by KS = 4/B symbols
//     (B = bits per symbol), entry = dest << 11 | lane << 2 | hits << 28, replicated per lane
//     so lane l always reads bank l (conflict-free).  Next offset = (e & 0xFFFF) | group << 7:
//     one LOP3, one LDS, one LEA.HI per group and route;
//   * tab1[s][c] = dest | acc << 15 for single-symbol steps (unaligned heads and tails) and
//     for the generic path (A > 4).
#include <stdlib.h>

#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b0_t0_0(uint32_t K);
const void* tiny_dispatch_b0_t1_0(uint32_t K);
const void* tiny_dispatch_b0_t1_1(uint32_t K);
const void* tiny_dispatch_b1_t0_0(uint32_t K);
const void* tiny_dispatch_b1_t1_0(uint32_t K);
const void* tiny_dispatch_b1_t1_1(uint32_t K);
const void* tiny_dispatch_b2_t0_0(uint32_t K);
const void* tiny_dispatch_b2_t1_0(uint32_t K);
const void* tiny_dispatch_b2_t1_1(uint32_t K);

namespace {

const void* tiny_dispatch(uint32_t K, uint32_t B, bool tma) {
    const void* f = nullptr;
    const uint32_t T = tma ? 1u : 0u;
    if (!f && B == 0 && T == 0) f = tiny_dispatch_b0_t0_0(K);
    if (!f && B == 0 && T == 1) f = tiny_dispatch_b0_t1_0(K);
    if (!f && B == 0 && T == 1) f = tiny_dispatch_b0_t1_1(K);
    if (!f && B == 1 && T == 0) f = tiny_dispatch_b1_t0_0(K);
    if (!f && B == 1 && T == 1) f = tiny_dispatch_b1_t1_0(K);
    if (!f && B == 1 && T == 1) f = tiny_dispatch_b1_t1_1(K);
    if (!f && B == 2 && T == 0) f = tiny_dispatch_b2_t0_0(K);
    if (!f && B == 2 && T == 1) f = tiny_dispatch_b2_t1_0(K);
    if (!f && B == 2 && T == 1) f = tiny_dispatch_b2_t1_1(K);
    return f;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = []() -> EncodeFn {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

}  // namespace

// A 2-D uint8 tensor map over rows of `row_len` bytes (row stride = row_len), box
// box_w x box_rows, 64-byte swizzle (TMA row streaming: tiny kernel, converging follow).
bool encode_rows_map(CUtensorMap* map, const uint8_t* base, uint64_t row_len, uint64_t rows, uint32_t box_w,
                     uint32_t box_rows) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)row_len, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)row_len};
    const cuuint32_t box[2] = {box_w, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Register slots per chunk (routes advanced together).  Generic-alphabet kernels (B = 0:
// one table lookup per symbol) are instantiated for fewer K to bound the build.
uint32_t tiny_round_slots(uint32_t k, uint32_t B) {
    static const uint32_t ks[] = {1, 2, 3, 4, 6, 8, 12, 16};
    static const uint32_t k0[] = {1, 2, 4, 8};
    if (B == 0) {
        for (uint32_t v : k0)
            if (k <= v) return v;
        return 8;   // more candidates: extra passes over the chunk
    }
    for (uint32_t v : ks)
        if (k <= v) return v;
    return 16;
}

size_t tiny_smem_bytes(const DevDfa& d, uint32_t B, uint32_t stages) {
    return tiny_layout(d.Qp, d.Qpad, d.A, d.Lsum_all, B, stages).total;
}

// TMA stages per warp: two 4 KB boxes (16 warps x 2 = 32 boxes in flight per SM; more than
// ~48 collapses TMA throughput and 3 stages measured 1.8% slower on cfg2,
// profiles/r01_stream_probe.txt), fewer if the tables leave no room; 0 = no TMA staging.
uint32_t tiny_pick_stages(const DevDfa& d, uint32_t B) {
    static int limit = 0;
    if (!limit) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0)
            v = 232448;
        limit = v;
    }
    uint32_t smax = 2;
    if (const char* e = getenv("PAREM_TINY_STAGES")) {   // experiments only (2 or 3)
        const int v = atoi(e);
        if (v >= 2 && v <= (int)kMaxStages) smax = (uint32_t)v;
    }
    for (uint32_t s = smax; s >= 2; --s)
        if (tiny_smem_bytes(d, B, s) <= (size_t)limit) return s;
    return 0;
}

int tiny_blocks_per_sm(uint32_t K, uint32_t B, bool tma, size_t smem) {
    const void* fn = tiny_dispatch(K, B, tma);
    if (!fn) return 0;
    smem_optin(fn, smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kT, smem) != cudaSuccess) return 0;
    return nb;
}

int launch_tiny(const Plan& plan, const MatchParams& P, cudaStream_t s) {
    // TMA staging needs a 16-B aligned input and rows of a multiple of the box width
    // (and every nominal row [t L, (t+1) L) inside the input: p L <= n)
    bool tma = plan.tma != 0 && (((uintptr_t)P.in) & 15u) == 0 && P.L % kBoxBytes == 0 && P.L >= kBoxBytes &&
               P.p * P.L <= P.n;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    if (tma) tma = encode_rows_map(&map, P.in, P.L, P.p, kBoxBytes, kRowsW);
    const void* fn = tiny_dispatch(plan.slots, P.d.sym_bits, tma);
    if (!fn) {
        set_error("no tiny kernel for K=%u B=%u", plan.slots, P.d.sym_bits);
        return PAREM_EINTERNAL;
    }
    MatchParams Q = P;
    Q.stages = tma ? plan.tma : 0u;
    const size_t smem = tiny_smem_bytes(P.d, P.d.sym_bits, Q.stages);
    cudaError_t e = smem_optin(fn, smem);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    void* args[] = {&Q, &map};
    e = cudaLaunchKernel(fn, dim3((unsigned)plan.grid), dim3(kT), args, smem, s);
    if (e != cudaSuccess) {
        set_error("tiny kernel launch: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    prof_after("tiny", s);
    return PAREM_OK;
}

}  // namespace parem
