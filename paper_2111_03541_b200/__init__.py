"""B200-native MetaFEM assembly path (arXiv:2111.03541): K x = d from PDE weak forms.

The product is libfem.so (csrc/, C ABI in include/libfem.h); `fem` is its ctypes binding and
`system` a small torch-tensor convenience layer on top of it.  No CPU fallback exists.
"""
from . import fem  # noqa: F401
from .system import FemSystem  # noqa: F401
