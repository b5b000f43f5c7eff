// me_box_k1_4.cu -- me_box instantiations for template sizes K in {1, 2, 3, 4} (a separate
// build unit of the kernels in me_box.cuh; launch_box in me_box.cu dispatches here).
#include "me_box.cuh"

namespace qs {
cudaError_t launch_box_k1_4(const BoxArgs &a, int K, bool ssd, bool reverse, cudaStream_t s) {
    switch (K) {
        case 1: return launch_k<1>(a, ssd, reverse, s);
        case 2: return launch_k<2>(a, ssd, reverse, s);
        case 3: return launch_k<3>(a, ssd, reverse, s);
        case 4: return launch_k<4>(a, ssd, reverse, s);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace qs
