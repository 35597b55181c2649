"""B200-native Jac-PCG RZF precoding (arxiv 2305.13925 hot path).

Reference-compatible entry points (same names as the reference package's
__init__.py:5-28 for the precoding path) plus batched device siblings.  All
arithmetic runs in libxlmimo_b200.so (hand-written sm_100a kernels); there is
no CPU fallback.
"""

__version__ = "0.1.0"

from .batched import (PrecoderBatch, apply_precoder_batched, combine_se_partials,  # noqa: F401
                      gram_batched, rzf_batched, se_partials, sinr_batched,
                      solve_batched, tensor_core_path, uses_tensor_cores)
from .channel import ChannelModel, beta_bar, build_correlation, generate_channels, psd_sqrt  # noqa: F401
from .configs import CONFIGS, Workload  # noqa: F401
from .errors import (AssemblyError, ConfigurationError, DegenerateChannelError,  # noqa: F401
                     GeometryInfeasibleError, ModelError, NotHpdError,
                     SplittingError, UnsupportedTopologyError, XlMimoError)
from .linsolve import (ITERATIVE_SOLVERS, HpdSystem, SolverOutcome, cg_solve,  # noqa: F401
                       direct_solve, gs_solve, jacpcg_solve, jor_solve)
from .metrics import LinkReport, coupling_matrix, sinr_eq9, sum_se  # noqa: F401
from .precoder import (BlockPrecoder, PrecoderBlock, assemble_precoder,  # noqa: F401
                       build_precoder, gram_regularized, rzf_block, rzf_direct,
                       rzf_iterative, solve_iterative)
