// Generation kernels of LIR-CMOP1-14 (problems.cpp:66-137): four sub-family kernels at d = 30.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

VaryKernel vary_kernel_lir(int mode, int op, int d, int id, bool tour) {
    if (d != 30 || mode != MODE_VARY) return pick_vary<EvalLir>(mode, op, tour);
    return id <= 4 ? pick_vary<EvalLirT<1>, 30, true>(mode, op, tour)
                   : (id <= 8 ? pick_vary<EvalLirT<5>, 30, true>(mode, op, tour)
                              : (id <= 12 ? pick_vary<EvalLirT<9>, 30, true>(mode, op, tour)
                                          : pick_vary<EvalLirT<13>, 30, true>(mode, op, tour)));
}

}  // namespace gmpea_b200
