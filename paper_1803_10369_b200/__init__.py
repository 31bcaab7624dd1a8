"""paper_1803_10369_b200 — B200-native SRLA engine (super points over sliding windows).

The product is libsrla_b200.so (csrc/, C ABI in include/srla.h); `srla` is its
Python host binding and `build` its sm_100a build recipe.
"""
from .srla import (  # noqa: F401
    DetectPipeline, DeviceTraceGenerator, ENTRY_DTYPE, EstimatorArray, PlantSpec, SeaConfig,
    INDICATOR, ROUGH, LINEAR, load_library, LIB_PATH,
)
