// Generation kernels of MW1-14 (restated) at d = 15.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

VaryKernel vary_kernel_mw(int mode, int op, int d, int id, bool tour) {
    (void)id;
    return d == 15 ? pick_vary<EvalMw, 15>(mode, op, tour) : pick_vary<EvalMw>(mode, op, tour);
}

}  // namespace gmpea_b200
