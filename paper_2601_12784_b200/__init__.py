"""StaleFlow (arXiv 2601.12784) staleness-constrained rollout-coordination step, B200-native.

The product is the sm_100a CUDA library behind include/staleflow.h; the Python
binding in `staleflow.py` only marshals arguments.  Import submodules
explicitly (`from paper_2601_12784_b200 import staleflow, workload`); this
package init loads nothing.
"""
__all__ = ["staleflow", "workload"]
