// kernels_tiny_inst_b0_t0.cu -- tiny kernel instantiations for B = 0 bits per symbol,
// TMA staging = false (one TU per (B, TMA) so the build compiles them in parallel).
#include "kernels_tiny_impl.cuh"

namespace parem {

const void* tiny_dispatch_b0_t0(uint32_t K) {
    switch (K) {
        case 1: return tiny_fn<1, 0, false>();
        case 2: return tiny_fn<2, 0, false>();
        case 3: return tiny_fn<3, 0, false>();
        case 4: return tiny_fn<4, 0, false>();
        case 6: return tiny_fn<6, 0, false>();
        case 8: return tiny_fn<8, 0, false>();
        case 12: return tiny_fn<12, 0, false>();
        case 16: return tiny_fn<16, 0, false>();
        default: return nullptr;
    }
}

}  // namespace parem
