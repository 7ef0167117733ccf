"""B200-native operator-representation inference (CMLCompiler path), drop-in for ``mlower``.

    import paper_2301_13441_b200 as cmlb
    compiled = cmlb.compile_model(cmlb.parse_model(json_text))
    y = cmlb.predict(compiled, x)            # x: host Tensor/ndarray or CUDA tensor
    y = cmlb.execute(mlower_plan, x)         # a reference KernelPlan runs unchanged

All compute runs in hand-written sm_100a kernels in ``libcmlb.so`` (C ABI:
``include/cmlb.h``); there is no CPU fallback.  See DESIGN.md.
"""

from .dtypes import DType
from .errors import MlowerError
from .models import parse_model
from .tensor import Tensor

__all__ = ["DType", "MlowerError", "Tensor", "parse_model", "compile_model", "predict", "execute",
           "from_plan", "CompileResult", "DEFAULT_TOLERANCE"]


def __getattr__(name):
    # torch-dependent API loads lazily so host-only tools (parsing, lowering)
    # stay importable without initialising CUDA
    if name in ("compile_model", "predict", "execute", "from_plan", "CompileResult", "DEFAULT_TOLERANCE"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
