// me_box_k5_9.cu -- me_box instantiations for template sizes K in {5, 6, 7, 9} (a separate
// build unit of the kernels in me_box.cuh; launch_box in me_box.cu dispatches here).
#include "me_box.cuh"

namespace qs {
cudaError_t launch_box_k5_9(const BoxArgs &a, int K, bool ssd, bool reverse, cudaStream_t s) {
    switch (K) {
        case 5: return launch_k<5>(a, ssd, reverse, s);
        case 6: return launch_k<6>(a, ssd, reverse, s);
        case 7: return launch_k<7>(a, ssd, reverse, s);
        case 9: return launch_k<9>(a, ssd, reverse, s);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace qs
