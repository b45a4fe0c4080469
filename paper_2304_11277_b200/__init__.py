"""B200-native FSDP runtime (arXiv 2304.11277 hot path).

Host-side layout/plan logic is importable anywhere; everything that touches
the device goes through the in-tree C-ABI library `_fsdp_b200.so`
(include/fsdp_b200.h) and raises ImportError if it has not been built —
there is no CPU fallback.
"""
from .layout import (FlatParamError, OriginalParam, SharedParameterError, UnitLayout,  # noqa: F401
                     build_unit_layouts, dump_plan_lines, peak_param_memory)
from .plan import CollectiveError, DeadlockError, ShardingPlan, build_plan  # noqa: F401

__version__ = "0.1.0"

_LAZY = {
    "FullyShardedDataParallel": "fsdp", "ShardingStrategy": "fsdp", "BackwardPrefetch": "fsdp",
    "MixedPrecision": "fsdp", "CPUOffload": "fsdp", "ModuleWrapPolicy": "fsdp",
    "transformer_auto_wrap_policy": "fsdp",
    "FSDPRuntime": "runtime", "RuntimeConfig": "runtime", "EngineError": "runtime",
    "StaticOrderError": "runtime", "RAF": "runtime", "NRAF": "runtime",
    "DeviceComm": "comm", "DeviceFabric": "comm",
    "Session": "session", "EngineConfig": "session", "PrecisionPolicy": "session",
    "ScalerConfig": "session", "ShardedGradScaler": "session", "ModelSpec": "session",
    "ACCUM_OFF": "session", "ACCUM_WITH_COMM": "session", "ACCUM_NO_COMM": "session",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
