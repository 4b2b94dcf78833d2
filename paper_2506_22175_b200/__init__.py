"""B200-native pipelined expert-parallel MoE layer (MPipeMoE, arxiv 2506.22175).

Data plane: hand-written sm_100a kernels in libmpm.so (include/mpm.h) —
tcgen05/TMEM/TMA grouped expert GEMMs (persistent, 2-CTA 256x256 tiles in a
static round-robin order), HBM-bound routing / permute / combine kernels (the
combine backward fused with the gate's softmax backward), and chunk exchanges
over NVLink peer memory (CUDA-IPC windows; senders gather their token rows
straight into the receivers' expert-side windows, one light copy kernel per
exchange, flags raised once per step and reset by their last waiter; grouped
NCCL send/recv as the explicitly selected baseline).  Control plane: a restatement of the reference planner
(`moepipesim`) whose schedule DAG is executed on CUDA streams by
runtime.PipelineExecutor.
"""

from .spec import (  # noqa: F401
    COLLECTIVE_STREAM, COMPUTE_STREAM, COPY_STREAM, STREAMS,
    BatchSpec, HardwareProfile, InvalidPartitioningError, ModelSpec, NO_REUSE, REUSE_STRATEGIES,
    RestoreMethod, ReuseNotApplicableError, ReuseStrategy, S1, S2, S3, S4, STRATEGIES, SlowdownTable,
    TensorRole, micro_batch_size,
)
from .memory import (  # noqa: F401
    MemoryReport, build_report, mem_activations_baseline, mem_buffers_baseline, mem_model_states,
    mem_pipeline, mem_reuse_savings, mem_saving_ratio,
)
from .cost import BaseVolumes, CostBreakdown, StrategySelection, base_volumes, select_strategy, stage_cost  # noqa: F401
from .schedule import OpNode, PoolSpec, ScheduleDag, ScheduleError, SlotSpec, build_schedule  # noqa: F401
from .granularity import (  # noqa: F401
    AdaptiveController, GranularityIndex, MeasurementAdapter, NoCandidateError, SearchStats, TrialBudget,
    generate_workload, noisy_adapter, search_best_gran,
)
from .trace import (  # noqa: F401
    MemoryComponents, ScheduleTrace, TraceEvent, TraceInvariantError, exposed_a2a_fraction,
    memory_components, peak_memory, replay_validate, to_jsonl, to_trace_event, write_trace,
)


def __getattr__(name):
    # torch-dependent symbols load lazily so the planner imports without CUDA
    if name in ("MoELayer",):
        from .layer import MoELayer
        return MoELayer
    raise AttributeError(name)
