"""B200-native executor for HexiScale's asymmetric-parallel training step.

The product is the C-ABI library libhexexec.so (include/hexexec.h); this
package is the Python-side mirror of that interface (ctypes), used by the
tests, bench.py and torch.distributed bootstrap.  Importing it loads the
library and fails loudly when it has not been built.
"""
from . import _lib  # noqa: F401  (raises ImportError when the .so is missing)
from .hexexec import Executor, Plan, HexexecError  # noqa: F401

__all__ = ["Executor", "Plan", "HexexecError"]
