// kernels_tiny_inst_b0_t1_1.cu -- tiny kernel instantiations for B = 0 bits per symbol,
// TMA staging = true, register slots K in {4, 8} (one TU per group so the
// build compiles the register-unrolled variants in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b0_t1_1(uint32_t K) {
    switch (K) {
        case 4: return tiny_fn<4, 0, true>();
        case 8: return tiny_fn<8, 0, true>();
        default: return nullptr;
    }
}

}  // namespace parem
