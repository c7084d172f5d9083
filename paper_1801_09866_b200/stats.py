"""Host-side reporting formulas of the paper's cache statistics."""
from __future__ import annotations


def redundancy_rate(baseline_count: int, quantized_count: int) -> float:
    """Table 1's "Redundancy rate": (baseline - quantized) / baseline * 100,
    reported to two decimals."""
    if baseline_count <= 0:
        raise ValueError("redundancy rate undefined for a zero baseline")
    if not 0 <= quantized_count <= baseline_count:
        raise ValueError("need baseline >= quantized >= 0")
    return round((baseline_count - quantized_count) / baseline_count * 100.0, 2)


def hit_ratio(hits: int, lookups: int) -> float:
    """Cache hit ratio, "around 89%" for the LM-query cache."""
    if lookups <= 0:
        raise ValueError("hit ratio undefined without lookups")
    return hits / lookups
