// kernels_tiny_inst_b0_t1_0.cu -- tiny kernel instantiations for B = 0 bits per symbol,
// TMA staging = true, register slots K in {1, 2} (one TU per group so the
// build compiles the register-unrolled variants in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b0_t1_0(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 0, true>();
        case 2: return tiny_fn<2, 0, true>();
        default: return nullptr;
    }
}

}  // namespace parem
