"""B200-native executor for HydraInfer's data-parallel serving hot path.

Drops in under the reference scheduler (``epdsim``): the reference's stage-level
batching, admission, routing and migration protocol run unchanged, and every batch /
migration they produce executes on sm_100a kernels from ``libhydra_sm100.so``.

Public API
  GpuCluster, run_trace_gpu      drop-in for epdsim.Cluster / run_trace
  GpuMigrationJob                drop-in for epdsim.MigrationJob (S3)
  PhysicalCachePool              drop-in for epdsim.engine.CachePool (S2)
  InstanceRuntime                per-instance device state + batch executor (S1)
  MllmShape, PRESETS, get_shape  executed model shapes (tiny, llava-1.5-7b, qwen2-vl-7b)
  b200_hardware                  HardwareProfile for one B200
"""

from . import _lib  # noqa: F401  (the .so loads on first device use: GpuCluster,
#                     InstanceRuntime, DeviceWeights; a missing library raises there --
#                     there is no CPU fallback -- while the host-only modules (shapes,
#                     inputs, planner) stay importable without mapping it)

from ._epdsim import E as epdsim  # noqa: E402
from .shapes import MllmShape, PRESETS, get_shape, with_layers  # noqa: E402
from .pools import PhysicalCachePool  # noqa: E402


def b200_hardware(peak_flops: float = 2.25e15, mem_bandwidth: float = 8.0e12,
                  gpu_memory_bytes: float = 160e9, model_weight_bytes: float = 14e9,
                  interconnect_bandwidth: float = 900e9):
    """A B200 ``HardwareProfile`` (model_cost.py:66-86).  ``gpu_memory_bytes`` is set
    below the 183 GB physical so the pools sized by ``pool_capacities`` plus weights and
    workspaces fit on the device; the scheduler and the executor use the same value."""
    return epdsim.HardwareProfile(peak_flops, mem_bandwidth, gpu_memory_bytes,
                                  model_weight_bytes, interconnect_bandwidth)


def __getattr__(name):
    if name in ("GpuCluster", "GpuMigrationJob", "run_trace_gpu", "batch_log_digest"):
        from . import cluster
        return getattr(cluster, name)
    if name == "InstanceRuntime":
        from .executor import InstanceRuntime
        return InstanceRuntime
    raise AttributeError(name)


__all__ = ["GpuCluster", "GpuMigrationJob", "run_trace_gpu", "batch_log_digest",
           "PhysicalCachePool", "InstanceRuntime", "MllmShape", "PRESETS", "get_shape",
           "with_layers", "b200_hardware", "epdsim"]
