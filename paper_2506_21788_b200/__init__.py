"""B200-native multi-task-parallel GNN training step (arxiv 2506.21788 hot path).

The compute lives in libhmtl_b200.so (hand-written sm_100a CUDA behind the C ABI
in include/hmtl_b200.h); this package is the thin host-side mirror of the
reference's C++ API used by tests and the benchmark.
"""
from ._lib import HmtlError, build, lib  # noqa: F401
from .model import (  # noqa: F401
    Caps, GradientBufferT, checkpoint_hyper, checkpoint_write, GraphBatch, ModelHyper, ModelT, PredictionT, Samples, SampleStore, TrainConfig,
    align_energies, classify_regime, comm_unique_id, epoch_plan, make_partition, shard_range, head_layout, hmtd_header, hmtd_write, memory_footprint, nbr_build, shared_layout,
)
