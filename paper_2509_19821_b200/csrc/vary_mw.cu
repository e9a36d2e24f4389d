// Generation kernels of MW1-14 (restated) at d = 15.
#include "vary_dispatch.cuh"

namespace gmpea_b200 {

#ifndef GMPEA_PER_PROBLEM
#define GMPEA_PER_PROBLEM 1  // SBX generation kernels compiled per MW problem (A/B switch)
#endif

template <int ID>
static VaryKernel mw_sbx() {
    return vary_eval_kernel<EvalMwT<ID>, MODE_VARY, OP_SBX, 15, true>;
}

VaryKernel vary_kernel_mw(int mode, int op, int d, int id, bool tour) {
    // the suite's operator (SBX) at d = 15: one kernel per problem
    if (GMPEA_PER_PROBLEM && d == 15 && mode == MODE_VARY && op == OP_SBX && !tour) {
        switch (id) {
            case 1: return mw_sbx<1>();
            case 2: return mw_sbx<2>();
            case 3: return mw_sbx<3>();
            case 4: return mw_sbx<4>();
            case 5: return mw_sbx<5>();
            case 6: return mw_sbx<6>();
            case 7: return mw_sbx<7>();
            case 8: return mw_sbx<8>();
            case 9: return mw_sbx<9>();
            case 10: return mw_sbx<10>();
            case 11: return mw_sbx<11>();
            case 12: return mw_sbx<12>();
            case 13: return mw_sbx<13>();
            case 14: return mw_sbx<14>();
            default: break;
        }
    }
    return d == 15 ? pick_vary<EvalMw, 15>(mode, op, tour) : pick_vary<EvalMw>(mode, op, tour);
}

}  // namespace gmpea_b200
