"""B200-native embedding lookup+update hot path of Persia (arXiv 2111.05897).

The product is ``libhps.so`` (CUDA kernels for sm_100a behind the C ABI in
``include/hps_c.h``); :mod:`.hps` is the Python host mirror of the reference's
PsShard / ShardSet / EmbeddingWorker operator API, :mod:`.workloads` generates the
synthetic batches of BASELINE.json's configs.
"""
from . import hps  # noqa: F401
from .hps import (ADAGRAD, MEAN, SGD, SUM, EmbeddingWorker, ShardSet, compress_indices,  # noqa: F401
                  dedup, mix64, route_shard)
