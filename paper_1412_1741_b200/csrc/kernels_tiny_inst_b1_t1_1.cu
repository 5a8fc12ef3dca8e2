// kernels_tiny_inst_b1_t1_1.cu -- tiny kernel instantiations for B = 1 bits per symbol,
// TMA staging = true, register slots K in {6, 8, 12, 16} (one TU per group so the
// build compiles the register-unrolled variants in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b1_t1_1(uint32_t K) {
    switch (K) {
        case 6: return tiny_fn<6, 1, true>();
        case 8: return tiny_fn<8, 1, true>();
        case 12: return tiny_fn<12, 1, true>();
        case 16: return tiny_fn<16, 1, true>();
        default: return nullptr;
    }
}

}  // namespace parem
