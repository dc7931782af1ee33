"""B200-native SSE electron self-energy (drop-in for negflow.sse.sse_sigma).

Hot path: Sigma^{<>} of the NEGF Born loop's SSE phase (reference
/root/reference/pkg/src/negflow/sse.py:305-329) on sm_100a FP64 tensor cores,
behind the C ABI in include/sse.h (libsse.so).  See DESIGN.md.
"""

from .types import (
    CombinedD,
    EnergyGrid,
    FlopCounter,
    GreensTensor,
    NeighborMap,
    SelfEnergyTensor,
    SimParams,
    SseVariant,
    build_neighbor_map,
    default_grid,
)
from .sse import alg_flops, pi_tallies, sigma_tallies, sse_pi, sse_sigma

__version__ = "0.1.0"

__all__ = [
    "CombinedD",
    "EnergyGrid",
    "FlopCounter",
    "GreensTensor",
    "NeighborMap",
    "SelfEnergyTensor",
    "SimParams",
    "SseVariant",
    "alg_flops",
    "build_neighbor_map",
    "default_grid",
    "pi_tallies",
    "sigma_tallies",
    "sse_pi",
    "sse_sigma",
]
