"""paper_2306_02526_b200: B200-native (sm_100a) drop-in for the per-stage HPS
solve path of arXiv 2306.02526's reference package ``hpstep``.

The public names mirror ``hpstep`` (pkg/src/hpstep/__init__.py) for the hot
path: tree numbering, coefficients / discretization, the HPS operator set
(build + solves on the GPU) and the IMEX ARK time stepper.
"""

from .chebyshev import ChebGrid1D, cheb_nodes, diff_matrix
from .errors import (ConfigError, DivergenceError, HpstepError, InvalidStepError,
                     SingularMatrixError, UnknownTableauError, UnsupportedConfigurationError)
from .operators import (EllipticDiscretization, LeafStencil, OperatorCoefficients, leaf_matrix,
                        shift_reaction)
from .solver import HpsOperatorSet, build, build_leaf, merge
from .tableaux import ButcherPair, available_tableaux, load_tableau
from .timestep import (ParabolicProblem, SeparableField, StepperState, TimeStepper,
                       declare_nonlinear, evaluate_nonlinear, gradient_use, is_pure,
                       scalar_stability_function)
from .tree import DomainTree, TreeNode, build_tree
from .stability import StepMapSpectrum, analyze, assemble_step_map
from .sharding import ShardedTimeStepper

__version__ = "0.1.0"

__all__ = [
    "ChebGrid1D", "cheb_nodes", "diff_matrix", "ConfigError", "DivergenceError", "HpstepError",
    "InvalidStepError", "SingularMatrixError", "UnknownTableauError",
    "UnsupportedConfigurationError", "EllipticDiscretization", "LeafStencil",
    "OperatorCoefficients", "leaf_matrix", "shift_reaction", "HpsOperatorSet", "build",
    "build_leaf", "merge", "scalar_stability_function", "DomainTree",
    "TreeNode", "build_tree", "ButcherPair", "available_tableaux", "load_tableau",
    "ParabolicProblem", "SeparableField", "StepperState", "TimeStepper", "evaluate_nonlinear",
    "declare_nonlinear", "gradient_use", "is_pure",
    "StepMapSpectrum", "analyze", "assemble_step_map", "ShardedTimeStepper",
]
