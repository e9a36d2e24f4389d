// Generation kernels of C/DC-DTLZ (problems.cpp:141-201, 409-527) at d = 7 / 12.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

VaryKernel vary_kernel_dtlz(int mode, int op, int d, int id, bool tour) {
    (void)id;
    return d == 7 ? pick_vary<EvalDtlz, 7>(mode, op, tour)
                  : (d == 12 ? pick_vary<EvalDtlz, 12>(mode, op, tour) : pick_vary<EvalDtlz>(mode, op, tour));
}

}  // namespace gmpea_b200
