// kernels_tiny_inst_b2_t0_0.cu -- tiny kernel instantiations for B = 2 bits per symbol,
// TMA staging = false, register slots K in {1, 2, 3, 4, 6, 8, 12, 16} (one TU per group so the
// build compiles the register-unrolled variants in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b2_t0_0(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 2, false>();
        case 2: return tiny_fn<2, 2, false>();
        case 3: return tiny_fn<3, 2, false>();
        case 4: return tiny_fn<4, 2, false>();
        case 6: return tiny_fn<6, 2, false>();
        case 8: return tiny_fn<8, 2, false>();
        case 12: return tiny_fn<12, 2, false>();
        case 16: return tiny_fn<16, 2, false>();
        default: return nullptr;
    }
}

}  // namespace parem
