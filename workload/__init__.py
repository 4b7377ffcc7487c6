"""Seeded synthetic workload generators shared by tests, bench and the oracle legs.

Holds none of the method's arithmetic (no routing, scoring, partitioning):
only random draws shaped like the paper's workloads and
the north_star's bimodal / heavy-tailed mixes.  Recipes are stated in
DESIGN.md §4.
"""
from .gen import (  # noqa: F401
    bimodal, heavy, lengths, arrivals, cost_estimates, pool, shard_range,
    THETA0, random_thetas, quantile_bounds, NOW, DEFAULT_COST,
)
