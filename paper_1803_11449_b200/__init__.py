"""B200-native super point detector hot path (arXiv 1803.11449, double-direction hash).

Scan -> per-cell estimate -> restore -> re-estimate + threshold filter as
hand-written sm_100a kernels behind a C ABI (include/dhsa_b200.h), with the
reference package's detector API on top:

    from paper_1803_11449_b200 import DhgParams, Dhla
    sketch = Dhla(DhgParams())              # 10 MiB of HBM at the defaults
    sketch.update_batch(src, dst)            # numpy (staged) or torch CUDA tensors (in place)
    reports = sketch.restore_superpoints(1024)

There is no CPU implementation in this package: without the CUDA library or a
GPU every data-path call raises.
"""

from . import dhg
from .dhg import DhgParams
from .dhla import (DEFAULT_MAX_CANDIDATES, Dhla, Estimate, SuperPointReport, hot_threshold,
                   merge, release_cached)
from .engine import (DetectionEngine, TRACE_DTYPE, WindowConfig, WindowResult, WindowSession,
                     split_pairs)
from .exact import EvalMetrics, ExactCounter, evaluate, exact_oracle
from .traces import GeneratorConfig, generate_trace, generate_trace_device
from .snapshot import read_snapshot, write_snapshot
from .errors import (CapacityError, ConfigError, CudaError, DataError, DhsaError,
                     SealedWindowError)

__version__ = "0.2.0"

__all__ = [
    "DhgParams", "dhg", "Dhla", "SuperPointReport", "Estimate", "merge", "hot_threshold", "release_cached",
    "DEFAULT_MAX_CANDIDATES", "DetectionEngine", "WindowConfig", "WindowResult", "WindowSession",
    "split_pairs", "TRACE_DTYPE", "read_snapshot", "write_snapshot", "GeneratorConfig", "generate_trace", "generate_trace_device", "exact_oracle", "ExactCounter", "evaluate", "EvalMetrics", "DhsaError", "ConfigError", "DataError", "CapacityError",
    "SealedWindowError", "CudaError",
]
