// kernels_tiny_inst_b2_t1.cu -- tiny kernel instantiations for B = 2 bits per symbol,
// TMA staging = true (one TU per (B, TMA) so the build compiles them in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b2_t1(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 2, true>();
        case 2: return tiny_fn<2, 2, true>();
        case 3: return tiny_fn<3, 2, true>();
        case 4: return tiny_fn<4, 2, true>();
        case 6: return tiny_fn<6, 2, true>();
        case 8: return tiny_fn<8, 2, true>();
        case 12: return tiny_fn<12, 2, true>();
        case 16: return tiny_fn<16, 2, true>();
        default: return nullptr;
    }
}

}  // namespace parem
