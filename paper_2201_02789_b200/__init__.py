"""B200-native nested-parallel hot path of arXiv 2201.02789 (CDP2 + thresholding,
coarsening and aggregation), behind the reference's ``dynoptc.bench`` API."""

__version__ = "0.1.0"
