"""B200-native spatial-coalescing hot path of the OoO VLIW JIT (arXiv 1901.10008).

Drop-in for the `gpumux` decision API (coalesce / scheduler / kernels /
device / tuning lookup), backed by a native C++ decision core, plus the thing
the reference only simulates: `Executor`, one persistent sm_100a launch per
scheduler step whose tile work list spans every member of every superkernel
dispatched in that step (tcgen05/TMEM grouped GEMM, streaming GEMV and
elementwise work items).
"""

from .coalesce import (DEFAULT_PAD_BUDGET, ShapeCluster, SuperKernel, cluster_shapes,
                       form_superkernel, pad_cost)
from .device import (CostEstimate, DeviceProfile, ProfileError, load_profile,
                     occupancy_efficiency, op_byte_ratio, roofline_duration)
from .kernels import (NO_DEADLINE, InferenceRequest, KernelSpec, LatencyConstraint,
                      block_count, bytes_moved, flop_count, kernel_cost, lower_model, submit)
from .scheduler import (CompletionInfo, Dispatch, EvictionRecord, PolicyParams, Scheduler,
                        SchedulerPolicy, TimelineEntry, slack)
from .tuning import DEFAULT_CONFIG, ClusterKey, TuningConfig, TuningTable

__version__ = "0.1.0"


def __getattr__(name):
    # the executor pulls in torch + the CUDA library; load it lazily
    if name in ("Executor", "OperandSet"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
