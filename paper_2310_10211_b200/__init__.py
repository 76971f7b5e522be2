"""B200-native fitness evaluator for GEVO-ML (arXiv 2310.10211).

Drop-in for the reference's evaluation hot path (`evotir`):
  _Evaluator / evaluate / holdout_report   -> shims.GpuEvaluator / evaluate / holdout_report
  nondominated_sort / crowding_distance /
  rank_population / select_survivors       -> shims (libgevo NSGA-II kernels)
Device work runs in libgevo.so (csrc/, include/gevo.h); this package is the
host side: program reader (dialect), lowering (lowering, plan), workloads,
evaluator, shims and the multi-GPU sharding (distributed).
"""
__version__ = "0.1.0"
