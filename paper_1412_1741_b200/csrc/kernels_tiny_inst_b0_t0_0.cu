// kernels_tiny_inst_b0_t0_0.cu -- tiny kernel instantiations for B = 0 bits per symbol,
// TMA staging = false, register slots K in {1, 2, 4, 8} (one TU per group so the
// build compiles the register-unrolled variants in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b0_t0_0(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 0, false>();
        case 2: return tiny_fn<2, 0, false>();
        case 4: return tiny_fn<4, 0, false>();
        case 8: return tiny_fn<8, 0, false>();
        default: return nullptr;
    }
}

}  // namespace parem
