"""pm4g: B200-native hot path of PM4Py-GPU (arXiv 2204.04898).

The product is libpm4g.so (C ABI, include/pm4g.h) built from csrc/ for sm_100a;
``pm4g`` is its thin ctypes binding.
"""
from . import pm4g  # noqa: F401
from .pm4g import Log, VariantTable, pm4g_log_create, Pm4gError  # noqa: F401
