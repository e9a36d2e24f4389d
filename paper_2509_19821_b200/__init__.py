"""GMPEA on B200: host-side mirror of the reference's Problem / Algorithm /
operator interfaces over the engine's C ABI (include/gmpea_b200.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/gmpea/*.hpp):

  make_problem / problem_names / make_wta_problem     problems.hpp:19-45, wta.hpp
  evaluate / evaluate_population                      problems.hpp:47-51, gmpea.hpp:33
  reference_vectors / build_neighborhoods             gmpea.hpp:37-51
  reproduce                                           gmpea.hpp:56-73
  environmental_selection                             gmpea.hpp:75-111
  igd / hypervolume / metric_front                    metrics.hpp:15-29
  RunConfig / GenRecord / RunResult / run_gmpea       gmpea.hpp:113-144

std::invalid_argument surfaces as ValueError, std::runtime_error as
RuntimeError.  All compute runs on the GPU through libgmpea_b200.so; there is
no CPU fallback — importing the package fails if the library is missing.
"""
from __future__ import annotations

from ._lib import (  # noqa: F401
    GMPEA_OP_DE,
    GMPEA_OP_SBX_PM,
    Engine,
    EvalResult,
    GenRecord,
    NeighborhoodTopology,
    OperatorParams,
    Population,
    Problem,
    RunConfig,
    RunResult,
    SelectionContext,
    Aggregation,
    VariationOp,
    build_neighborhoods,
    crowding_distance,
    environmental_selection,
    evaluate,
    evaluate_population,
    hypervolume,
    igd,
    lattice_neighborhoods,
    lib_path,
    make_problem,
    make_wta_problem,
    metric_front,
    nccl_unique_id,
    nondominated_sort,
    pf_reference,
    problem_names,
    reference_vectors,
    reproduce,
    run_baseline,
    run_gmpea,
    spea2_fitness,
    spea2_select,
)

__all__ = [n for n in dir() if not n.startswith("_")]
