"""B200-native quantum-trajectory (Monte Carlo wave-function) engine.

Drop-in for the data-parallel hot path of the reference package ``mcwf``
(arXiv:1810.03047, QTM): integrate many independent trajectories under
G = -i H_eff with quantum jumps, and average expectation values over the
ensemble -- on the GPU, behind the C ABI in include/qtm.h.  Both ODE
method families (ADAMS, BDF) and time-dependent Hamiltonians
H(t) = H0 + sum_k c_k(t) H_k (TimeDependentGenerator) run on the device.

    from paper_1810_03047_b200 import run_gpu, configs
    result = run_gpu(configs.build("c4"), 4096, 987654321)

Host-side types mirror the reference API (QuantumProblem, OdeConfig,
TrajectoryResult, OdeFailure, CsrMatrix, operator constructors); the
reference's own problem objects are accepted unchanged.
"""

from .csr import CsrMatrix, dagger, tensor, to_csr
from .engine import (DeviceProblem, partition_trajectories, raise_for_status, run_gpu,
                     run_sharded)
from .packing import PackedProblem, pack_problem
from .problem import (ADAMS, BDF, OdeConfig, OdeFailure, QuantumProblem, RunOptions,
                      TrajectoryResult, adams_tables, auto_step, average_trajectories, bdf_tables)
from .timedep import Coefficient, TimeDependentGenerator
from .qops import (EffectiveGenerator, OperatorSet, coherent, destroy, effective_generator, eye,
                   fock, sigma_minus, sigma_x, sigma_z)
from . import configs

DEFAULT_SEED = 987654321  # reference rng.py:25

__version__ = "0.1.0"
