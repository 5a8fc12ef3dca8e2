// kernels_segment.cu -- SURVEY §8(e): one input sharded over G GPUs.  The paper splits T
// into parts processed independently and joins their routes; a GPU
// that holds segment g > 0 of T does not know its entering state either, so it computes
// its segment's MAP over the paper's candidate set R = L(last byte of segment g-1) (P:67,
// P:84-99; S = Q for complete tables): every r in R -> (end state, match count).  The G
// maps are all-gathered (one collective) and folded along q0's path (parem_fold_segment_maps).
//
// Device side here: the multi-start HEAD walk -- every candidate walks the first X bytes of
// the segment (thread per candidate, the warp's lanes read the same byte: broadcast loads),
// recording its state at X and its hits.  Routes merge (Table II), so the X-states
// collapse to a few distinct states z; the host then finishes each z over [X, n) with one
// ordinary match (parem_match_continue_async) and combines (abi.cu, parem_segment_map).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels_common.cuh"

namespace parem {

namespace {

__global__ void __launch_bounds__(256) segment_head_kernel(const DevDfa d, const uint8_t* __restrict__ in, uint64_t X,
                                                           const uint32_t* __restrict__ cand, uint32_t ncand,
                                                           uint32_t* __restrict__ st_out,
                                                           unsigned long long* __restrict__ hits_out,
                                                           unsigned long long* __restrict__ bad_inv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < ncand;
    uint32_t s = live ? cand[i] : 0u;
    unsigned long long h = 0;
    uint32_t badseen = 0;
    const bool tiny = d.tab1 != nullptr;
    const uint32_t ES = d.lanes_u32 ? 4u : 2u, ACC = d.lanes_u32 ? 31u : 15u;
    const uint32_t COL = d.Qpad * ES, SMASK = (d.Qpad - 1u) * ES;
    const unsigned char* g = reinterpret_cast<const unsigned char*>(d.lanes_tab);
    uint32_t e = s * ES;
    for (uint64_t k = 0; k < X; ++k) {
        uint32_t c = __ldg(in + k);   // same address in every lane: one broadcast transaction
        badseen |= c >= d.A;
        if (c >= d.A) c = d.A - 1;    // ESYMBOL is reported; keep the walk inside the table
        if (tiny) {
            const uint32_t t = __ldg(d.tab1 + s * d.A + c);
            s = t & 0x7FFFu;
            h += t >> 15;
        } else {
            const uint32_t off = (e & SMASK) + c * COL;
            e = d.lanes_u32 ? __ldg(reinterpret_cast<const uint32_t*>(g + off))
                            : __ldg(reinterpret_cast<const uint16_t*>(g + off));
            h += e >> ACC;
        }
    }
    if (!tiny) s = (e & SMASK) / ES;
    if (live) {
        st_out[i] = s;
        hits_out[i] = h;
    }
    if (i == 0 && badseen) {
        for (uint64_t k = 0; k < X; ++k)
            if (__ldg(in + k) >= d.A) {
                atomicMax(bad_inv, ~(unsigned long long)k);
                break;
            }
    }
}

}  // namespace

int launch_segment_head(const DevDfa& d, const uint8_t* in, uint64_t X, const uint32_t* cand, uint32_t ncand,
                        uint32_t* st_out, unsigned long long* hits_out, unsigned long long* bad_inv, cudaStream_t s) {
    if (ncand == 0) return PAREM_OK;
    segment_head_kernel<<<(ncand + 255) / 256, 256, 0, s>>>(d, in, X, cand, ncand, st_out, hits_out, bad_inv);
    prof_after("segment_head", s);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("segment head kernel: %s", cudaGetErrorString(e));
        return PAREM_ECUDA;
    }
    return PAREM_OK;
}

}  // namespace parem
