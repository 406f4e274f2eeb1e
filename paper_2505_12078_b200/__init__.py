"""B200-native SPOCK: Chambolle-Pock + SuperMann/Anderson for scenario-tree
risk-averse optimal control, as a drop-in for the CP/SuperMann iteration of the
reference arxiv/paper_2505_12078 (proj/include/spock/solver.hpp).

The hot path (L, L*, the S1 tree sweeps, S2, S3, SuperMann/Anderson
reductions) runs as hand-written sm_100a CUDA kernels in
``_build/libspock_b200.so`` behind the C-ABI declared in
``include/spock_b200.h``; this package holds the host-side mirror of the
reference API (problem model, generators, ctypes solver).
"""
from .problem import (Box, ConePart, Raocp, RiskSpec, ScenarioTree, avar_spec, expectation_spec,
                      CONE_FREE, CONE_NONNEG, CONE_SOC, CONE_ZERO, RISK_AVAR, RISK_GENERAL)
from .rng import Philox
from .solver import SolveResult, SpockSolver

__all__ = ["Box", "ConePart", "Raocp", "RiskSpec", "ScenarioTree", "avar_spec", "expectation_spec",
           "Philox", "SpockSolver", "SolveResult", "CONE_FREE", "CONE_NONNEG", "CONE_SOC", "CONE_ZERO",
           "RISK_AVAR", "RISK_GENERAL"]
