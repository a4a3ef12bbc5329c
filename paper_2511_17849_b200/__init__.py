"""B200-native Pier optimizer hot path (arXiv 2511.17849).

Drop-in for the optimizer path of the reference package ``pier``: the inner
AdamW step, global-norm clipping, the lazy-start -> momentum-warmup ->
momentum-decay outer schedule and the Nesterov outer step, with the
reference's names (``pier/__init__.py:43-65``).  Compute runs in hand-written
sm_100a kernels behind the C-ABI library ``libpier_b200.so``
(include/pier_b200.h); the multi-GPU exchanges are hand-written kernels on
NVLink peer memory (the persistent AdamW || outer-exchange round, the sharded
lazy-phase step), one group per GPU, with NCCL for the ordering barriers and
communicator setup.  There is no CPU fallback.
"""

from .errors import ConfigError, NumericError, ProtocolError
from .optim import (AdamWConfig, AdamWState, MultiTensorAdamW, OuterState, ScheduleConfig, adamw_,
                    adamw_bf16_, adamw_step, clip_global_norm, fold_momentum, grad_sqnorm_,
                    grad_sqnorm_bf16_, inner_lr,
                    momentum_mu, norm_workspace, outer_lr, outer_step, outer_update_, pseudograd, read_clip,
                    warmup_fold_)
from .topology import (GroupComm, Topology, VirtualGroup, allreduce_avg, build_topology, concat_shards,
                       inner_gradient_sync, outer_delta_sync, padded_len, ring_allreduce_bytes, shard_offsets, shard_views)
from .offload import HostStore
from .engine import DILOCO_OUTER_LR, DILOCO_OUTER_MU, MODES, BoundaryRecord, CommStats, PierEngine, PierSchedule
from . import artifacts, desk, tinygpt  # noqa: F401  (reference artifact formats, GPU desk runs)
from .desk import (momentum_warmup_phase, run_adamw_baseline, run_diloco_baseline, run_pier,  # noqa: F401
                   run_training)

__version__ = "0.1.0"

__all__ = [
    "AdamWConfig", "AdamWState", "BoundaryRecord", "CommStats", "ConfigError", "DILOCO_OUTER_LR",
    "DILOCO_OUTER_MU", "GroupComm", "HostStore", "MODES", "MultiTensorAdamW", "NumericError", "OuterState",
    "PierEngine", "ProtocolError", "ScheduleConfig", "Topology", "VirtualGroup", "adamw_", "adamw_bf16_", "adamw_step",
    "allreduce_avg", "build_topology", "clip_global_norm", "concat_shards", "fold_momentum", "grad_sqnorm_", "grad_sqnorm_bf16_",
    "inner_gradient_sync", "inner_lr", "momentum_mu", "norm_workspace", "outer_delta_sync", "outer_lr",
    "outer_step", "outer_update_", "padded_len", "momentum_warmup_phase", "run_adamw_baseline",
    "run_diloco_baseline", "run_pier", "run_training", "pseudograd", "read_clip", "ring_allreduce_bytes",
    "shard_offsets", "shard_views", "warmup_fold_", "__version__",
]
