"""paper_2104_00237_b200 -- Optimizer Fusion (arXiv 2104.00237) on B200.

The reference's fused-optimizer API (/root/reference/pkg/src/optfuse/__init__.py:6-15)
over PyTorch modules, with every parameter update executed by hand-written
sm_100a multi-tensor kernels (``liboptfuse_b200.so``, C ABI in
``include/optfuse_b200.h``).  There is no CPU fallback: importing works
anywhere, but any update raises ``NativeLibraryError`` if the kernel library
is missing.
"""

from .errors import (ConfigError, GlobalInfoRequired, NativeLibraryError, NumericError,
                     SchedulingContractError, ShapeError, StateError)
from .graph import Graph, Layer, Parameter
from .models import build_classifier, build_model, iteration_inputs, make_input
from .engine import FusionEngine, launch_groups
from .optim import KINDS, OptimizerPolicy, clip_by_global_norm, newton_step
from .schedule import (BACKWARD_FUSION, BASELINE, FORWARD_FUSION, SCHEDULES,
                       StepReport, check_inplace_safety,
                       flush_pending_updates, run_backward_fusion, run_baseline,
                       run_forward_fusion)
from .trace import ScheduleTrace, critical_path_depth, validate_trace
from . import checkpoint  # noqa: E402  (state_dict / load_state_dict / observe)
from .graphs import CapturedStep

__version__ = "0.2.0"


def __getattr__(name):
    # torch.distributed is only imported when data parallel is asked for
    if name == "DataParallelFusion":
        from .dp import DataParallelFusion
        return DataParallelFusion
    raise AttributeError(name)
