// Generation kernels of C/DC-DTLZ (problems.cpp:141-201, 409-527) at d = 7 / 12.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

#ifndef GMPEA_PER_PROBLEM
#define GMPEA_PER_PROBLEM 1  // SBX generation kernels compiled per problem (A/B switch)
#endif

template <int ID, int DC>
static VaryKernel dtlz_sbx() {
    return vary_eval_kernel<EvalDtlzT<ID>, MODE_VARY, OP_SBX, DC, true>;
}

VaryKernel vary_kernel_dtlz(int mode, int op, int d, int id, bool tour) {
    // the suite's operator (SBX) at the registered dimensions (DTLZ1 shapes
    // d = 7, the others d = 12): one kernel per problem
    if (GMPEA_PER_PROBLEM && mode == MODE_VARY && op == OP_SBX && !tour) {
        if (d == 7) {
            switch (id) {
                case C1_DTLZ1: return dtlz_sbx<C1_DTLZ1, 7>();
                case DC1_DTLZ1: return dtlz_sbx<DC1_DTLZ1, 7>();
                case DC2_DTLZ1: return dtlz_sbx<DC2_DTLZ1, 7>();
                case DC3_DTLZ1: return dtlz_sbx<DC3_DTLZ1, 7>();
                default: break;
            }
        } else if (d == 12) {
            switch (id) {
                case C1_DTLZ3: return dtlz_sbx<C1_DTLZ3, 12>();
                case C2_DTLZ2: return dtlz_sbx<C2_DTLZ2, 12>();
                case C3_DTLZ4: return dtlz_sbx<C3_DTLZ4, 12>();
                case DC1_DTLZ3: return dtlz_sbx<DC1_DTLZ3, 12>();
                case DC2_DTLZ3: return dtlz_sbx<DC2_DTLZ3, 12>();
                case DC3_DTLZ3: return dtlz_sbx<DC3_DTLZ3, 12>();
                default: break;
            }
        }
    }
    return d == 7 ? pick_vary<EvalDtlz, 7>(mode, op, tour)
                  : (d == 12 ? pick_vary<EvalDtlz, 12>(mode, op, tour) : pick_vary<EvalDtlz>(mode, op, tour));
}

}  // namespace gmpea_b200
