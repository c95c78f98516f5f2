"""B200-native Anderson-accelerated Lloyd K-Means (arXiv 1805.10638).

The hot path (assignment, update, Anderson step) is hand-written sm_100a CUDA
behind the C ABI declared in ``include/aakm.h`` (``libaakm.so``).  This
package is the thin Python binding: argument marshalling only.  Importing it
does not load the CUDA library; :func:`paper_1805_10638_b200.aakm.lib` does,
and raises if it is missing (there is no CPU fallback).
"""
__all__ = ["aakm", "synthetic"]
