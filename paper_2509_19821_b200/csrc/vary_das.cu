// Generation kernels of DAS-CMOP1-9 (restated) at d = 30.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

#ifndef GMPEA_PER_PROBLEM
#define GMPEA_PER_PROBLEM 1  // SBX generation kernels compiled per problem (A/B switch)
#endif

template <int ID>
static VaryKernel das_sbx() {
    return vary_eval_kernel<EvalDasT<ID>, MODE_VARY, OP_SBX, 30, true>;
}

VaryKernel vary_kernel_das(int mode, int op, int d, int id, bool tour) {
    // the suite's operator (SBX) at d = 30: one kernel per problem (no problem
    // dispatch in the hot code: MW7 vary -11 %, MW1 -5 % for the MW family)
    if (GMPEA_PER_PROBLEM && d == 30 && mode == MODE_VARY && op == OP_SBX && !tour) {
        switch (id) {
            case 1: return das_sbx<1>();
            case 2: return das_sbx<2>();
            case 3: return das_sbx<3>();
            case 4: return das_sbx<4>();
            case 5: return das_sbx<5>();
            case 6: return das_sbx<6>();
            case 7: return das_sbx<7>();
            case 8: return das_sbx<8>();
            case 9: return das_sbx<9>();
            default: break;
        }
    }
    return d == 30 ? pick_vary<EvalDas, 30>(mode, op, tour) : pick_vary<EvalDas>(mode, op, tour);
}

}  // namespace gmpea_b200
