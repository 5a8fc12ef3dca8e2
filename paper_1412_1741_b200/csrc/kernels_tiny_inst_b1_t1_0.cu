// kernels_tiny_inst_b1_t1_0.cu -- tiny kernel instantiations for B = 1 bits per symbol,
// TMA staging = true, register slots K in {1, 2, 3, 4} (one TU per group so the
// build compiles the register-unrolled variants in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b1_t1_0(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 1, true>();
        case 2: return tiny_fn<2, 1, true>();
        case 3: return tiny_fn<3, 1, true>();
        case 4: return tiny_fn<4, 1, true>();
        default: return nullptr;
    }
}

}  // namespace parem
