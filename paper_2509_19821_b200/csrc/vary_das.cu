// Generation kernels of DAS-CMOP1-9 (restated) at d = 30.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

VaryKernel vary_kernel_das(int mode, int op, int d, int id, bool tour) {
    (void)id;
    return d == 30 ? pick_vary<EvalDas, 30>(mode, op, tour) : pick_vary<EvalDas>(mode, op, tour);
}

}  // namespace gmpea_b200
