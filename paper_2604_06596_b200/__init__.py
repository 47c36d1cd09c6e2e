"""B200-native DynLP batch update (arXiv 2604.06596) behind the reference API.

Public surface mirrors the reference package's update path
(/root/reference/pkg/src/dynlp/__init__.py): ``EngineConfig``,
``IterationReport``, ``BatchUpdate``, ``DynamicGraph``, ``LabelState``,
``apply_batch``, ``apply_batch_structure``, ``run_batches`` and
``itlp_batch_solve`` -- all executed by hand-written sm_100a CUDA kernels in
``libdynlp_b200.so`` through the C-ABI in ``include/dynlp_b200.h``.  The
native library is loaded on first use; if it is missing the call raises --
there is no CPU fallback.
"""

from .batch import BatchUpdate, EdgeList, read_batches_jsonl, write_batches_jsonl  # noqa: F401
from .errors import CudaError, FileFormatError, InternalError, ValidationError  # noqa: F401

__version__ = "0.1.0"

_ENGINE_NAMES = {
    "EngineConfig", "IterationReport", "DynamicGraph", "LabelState", "apply_batch",
    "apply_batch_structure", "run_batches", "itlp_batch_solve", "MODE_JACOBI",
    "MODE_GAUSS_SEIDEL", "DEFAULT_DELTA", "binary_label",
}


def __getattr__(name):
    if name in _ENGINE_NAMES:
        from . import engine

        return getattr(engine, name)
    raise AttributeError(name)
