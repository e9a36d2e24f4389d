// Generation kernels of weapon-target assignment (wta.cpp:51-129), streaming decode.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

VaryKernel vary_kernel_wta(int mode, int op, int d, int id, bool tour) {
    // id: 1 = more than kWtaNarrowSlots strike slots (64-bit decode keys)
    if (id)
        return d > 0 && mode == MODE_VARY ? pick_vary<EvalWtaT<true>, 0, true, true>(mode, op, tour)
                                          : pick_vary<EvalWtaT<true>>(mode, op, tour);
    return d > 0 && mode == MODE_VARY ? pick_vary<EvalWta, 0, true, true>(mode, op, tour)
                                      : pick_vary<EvalWta>(mode, op, tour);
}

}  // namespace gmpea_b200
