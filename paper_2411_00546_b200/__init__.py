"""B200-native (sm_100a, FP64) RASPEN hot path of the `ocp` package (arxiv 2411.00546).

Drop-in for the reference's ``raspen-eps`` path: the same entry points and
semantics as `pkg/src/ocp/schwarz.py` / `newton.py` / `krylov.py`, with every
per-subdomain and vector operation in hand-written CUDA kernels behind the C
ABI of ``include/ocp_gpu.h`` (``libocpgpu.so``).  See DESIGN.md.
"""

__version__ = "0.1.0"

from .grid import Grid, NonfiniteFieldError, build_laplacian, check_finite
from .system import (Cubic, ExpMinusOne, Nonlinearity, ProblemSpec, make_phi, merge_pair,
                     recover_control, smoothed_projection, smoothed_projection_derivative,
                     split_pair)
from .newton import (ContinuationSchedule, LinearSolveError, LineSearchError, NewtonConfig,
                     SolveReport, backtrack, newton_continuation)
from .krylov import GmresBreakdownError, GmresResult, KrylovConfig, gmres
from .schwarz import (CorrectionSet, Decomposition, LocalSolveError, Subdomain,
                      build_local_systems, decompose, local_correction, ras_fixed_point_step,
                      release_local_systems,
                      raspen_jacobian_apply, raspen_residual, raspen_solve)
from .engine import DeviceVector, Engine
from ._native import NativeError, NativeUnavailable
from .linear_ras import (GlobalJacobian, RasPreconditioner, global_jacobian, global_residual,
                         newton_ras_solve, ras_precondition, ras_preconditioner)
from .problem_setup import (StatePair, construct_plateau_problem, construct_test_problem,
                            solve_state)
from . import harness
