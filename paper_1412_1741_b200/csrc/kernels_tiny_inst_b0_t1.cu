// kernels_tiny_inst_b0_t1.cu -- tiny kernel instantiations for B = 0 bits per symbol,
// TMA staging = true (one TU per (B, TMA) so the build compiles them in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b0_t1(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 0, true>();
        case 2: return tiny_fn<2, 0, true>();
        case 3: return tiny_fn<3, 0, true>();
        case 4: return tiny_fn<4, 0, true>();
        case 6: return tiny_fn<6, 0, true>();
        case 8: return tiny_fn<8, 0, true>();
        case 12: return tiny_fn<12, 0, true>();
        case 16: return tiny_fn<16, 0, true>();
        default: return nullptr;
    }
}

}  // namespace parem
