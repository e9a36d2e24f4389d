// Generation-kernel instantiation per problem family.  Each vary_<family>.cu
// instantiates vary_eval_kernel for its evaluators (MODE_VARY / MODE_EVAL /
// MODE_INIT, SBX / DE, dimension-specialised where the suites fix d) so the
// families compile in parallel; engine.cu reaches them via vary_kernel_for.
#pragma once
#include "kernels.cuh"

namespace gmpea_b200 {

using VaryKernel = void (*)(VaryParams);

// the dimension-specialised generation kernels also assume uniform bounds
// (true of every registered suite; checked by the caller)
template <class Ev, int DC = 0, bool VARY_ONLY = false, bool UBF = false>
VaryKernel pick_vary(int mode, int op, bool tour = false) {
    if (tour) {  // the comparison algorithms: SBX children of tournament parents
        constexpr bool UBT = DC > 0 || UBF;
        return vary_eval_kernel<Ev, MODE_VARY, OP_SBX, DC, UBT, true>;
    }
    if (!VARY_ONLY) {
        if (mode == MODE_EVAL) return vary_eval_kernel<Ev, MODE_EVAL, OP_SBX>;
        if (mode == MODE_INIT) return vary_eval_kernel<Ev, MODE_INIT, OP_SBX>;
    }
    constexpr bool UB = DC > 0 || UBF;  // UBF: uniform bounds at a run-time dimension
    return op == OP_DE ? vary_eval_kernel<Ev, MODE_VARY, OP_DE, DC, UB> : vary_eval_kernel<Ev, MODE_VARY, OP_SBX, DC, UB>;
}


VaryKernel vary_kernel_lir(int mode, int op, int d, int id, bool tour);
VaryKernel vary_kernel_dtlz(int mode, int op, int d, int id, bool tour);
VaryKernel vary_kernel_wta(int mode, int op, int d, int id, bool tour);
VaryKernel vary_kernel_das(int mode, int op, int d, int id, bool tour);
VaryKernel vary_kernel_mw(int mode, int op, int d, int id, bool tour);

}  // namespace gmpea_b200
